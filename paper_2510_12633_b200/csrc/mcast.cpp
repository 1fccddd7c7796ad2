// NVSwitch multicast team of the LAM_HOP_MULTICAST broadcast (PAPER L1527:
// the bandwidth term M·T_byte is the floor of any broadcast — with NVLS the switch replicates every
// store, so the source's egress is M once and no relay forwards anything over NVLink).
//
// One multicast object; every team device (the actor GPU + every relay GPU) binds one "member"
// allocation of the same size.  Member layout = node 0's S slots (data, same offsets as node 0's
// part) followed by S chunk-flag arrays.  On the actor GPU the member IS node 0's slot data; on a
// relay GPU it is the local replica ("mirror") of node 0's slots that the relay's verify-and-commit
// hop reads from local HBM.  The pack stores through the multicast VA (multimem.st), which exists
// only in the process of the actor GPU.  The actor GPU's member is also handed to the other processes
// (mapped there): node 0's slot data is then a valid mapping in every process.
//
// Driver API through cudaGetDriverEntryPoint (the library does not link libcuda).  With one process
// per GPU the multicast handle (a POSIX file descriptor) travels from the actor's process to the
// others over an abstract unix socket (SCM_RIGHTS); cuMulticastBindMem blocks until every team
// device was added, so no extra barrier is needed.
#include <cuda.h>
#include <cuda_runtime.h>
#include <errno.h>
#include <poll.h>
#include <stdio.h>
#include <string.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <time.h>
#include <unistd.h>

#include "mcast.h"

namespace lam {
namespace {

struct Drv {
  CUresult (*create)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*add)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*bind)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                   unsigned long long) = nullptr;
  CUresult (*unbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*mc_gran)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
  CUresult (*mem_create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*mem_release)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*mem_gran)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*addr_free)(CUdeviceptr, size_t) = nullptr;
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*unmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*exp)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long) = nullptr;
  CUresult (*imp)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
  CUresult (*dev_get)(CUdevice*, int) = nullptr;
  CUresult (*attr)(int*, CUdevice_attribute, CUdevice) = nullptr;
  CUresult (*err_str)(CUresult, const char**) = nullptr;
  bool ok = false;
};

template <typename F>
bool sym(const char* name, F* fn) {
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess) {
    cudaGetLastError();
    return false;
  }
  *fn = reinterpret_cast<F>(p);
  return true;
}

const Drv& drv() {
  static Drv d = [] {
    Drv x;
    x.ok = sym("cuMulticastCreate", &x.create) && sym("cuMulticastAddDevice", &x.add) &&
           sym("cuMulticastBindMem", &x.bind) && sym("cuMulticastUnbind", &x.unbind) &&
           sym("cuMulticastGetGranularity", &x.mc_gran) && sym("cuMemCreate", &x.mem_create) &&
           sym("cuMemRelease", &x.mem_release) && sym("cuMemGetAllocationGranularity", &x.mem_gran) &&
           sym("cuMemAddressReserve", &x.reserve) && sym("cuMemAddressFree", &x.addr_free) &&
           sym("cuMemMap", &x.map) && sym("cuMemUnmap", &x.unmap) && sym("cuMemSetAccess", &x.access) &&
           sym("cuMemExportToShareableHandle", &x.exp) && sym("cuMemImportFromShareableHandle", &x.imp) &&
           sym("cuDeviceGet", &x.dev_get) && sym("cuDeviceGetAttribute", &x.attr) &&
           sym("cuGetErrorString", &x.err_str);
    return x;
  }();
  return d;
}

bool cu_ok(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return true;
  const char* s = "?";
  if (drv().err_str) drv().err_str(r, &s);
  fprintf(stderr, "liblam: multicast: %s failed: %s (%d)\n", what, s, (int)r);
  return false;
}

CUmemAllocationProp member_prop(int dev) {
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = dev;
  // an exported (shareable) multicast object binds only shareable memory
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return ap;
}

CUmulticastObjectProp mc_prop(int n_devices, uint64_t size) {
  CUmulticastObjectProp mp = {};
  mp.numDevices = (unsigned)n_devices;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = size;
  return mp;
}

uint64_t now_ms() {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (uint64_t)ts.tv_sec * 1000ull + (uint64_t)ts.tv_nsec / 1000000ull;
}

socklen_t sock_addr(const char* name, sockaddr_un* a) {
  memset(a, 0, sizeof *a);
  a->sun_family = AF_UNIX;
  // abstract namespace (leading NUL): nothing on the filesystem, gone with the last socket
  const size_t n = strnlen(name, sizeof a->sun_path - 2);
  memcpy(a->sun_path + 1, name, n);
  return (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + n);
}

// Owner: hand `fds` (the multicast object, the owner's member) to `n_peers` connecting processes
// (SCM_RIGHTS), waiting at most timeout_ms.
bool serve_fd(const char* name, const int fds[2], int n_peers, uint64_t timeout_ms) {
  int ls = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
  if (ls < 0) return false;
  sockaddr_un a;
  const socklen_t al = sock_addr(name, &a);
  if (bind(ls, (sockaddr*)&a, al) != 0 || listen(ls, 64) != 0) {
    fprintf(stderr, "liblam: multicast: socket %s: %s\n", name, strerror(errno));
    close(ls);
    return false;
  }
  const uint64_t t_end = now_ms() + timeout_ms;
  bool ok = true;
  for (int i = 0; i < n_peers && ok; ++i) {
    pollfd pf{ls, POLLIN, 0};
    const uint64_t t = now_ms();
    if (t >= t_end || poll(&pf, 1, (int)(t_end - t)) <= 0) {
      fprintf(stderr, "liblam: multicast: %d of %d processes never connected\n", n_peers - i, n_peers);
      ok = false;
      break;
    }
    int cs = accept(ls, nullptr, nullptr);
    if (cs < 0) { ok = false; break; }
    char byte = 'm';
    iovec io{&byte, 1};
    char ctrl[CMSG_SPACE(2 * sizeof(int))] = {};
    msghdr m = {};
    m.msg_iov = &io;
    m.msg_iovlen = 1;
    m.msg_control = ctrl;
    m.msg_controllen = sizeof ctrl;
    cmsghdr* cm = CMSG_FIRSTHDR(&m);
    cm->cmsg_level = SOL_SOCKET;
    cm->cmsg_type = SCM_RIGHTS;
    cm->cmsg_len = CMSG_LEN(2 * sizeof(int));
    memcpy(CMSG_DATA(cm), fds, 2 * sizeof(int));
    ok = sendmsg(cs, &m, 0) == 1;
    close(cs);
  }
  close(ls);
  return ok;
}

// Peer: receive the owner's two descriptors (retrying until the owner listens).
bool fetch_fd(const char* name, uint64_t timeout_ms, int fds[2]) {
  const uint64_t t_end = now_ms() + timeout_ms;
  sockaddr_un a;
  const socklen_t al = sock_addr(name, &a);
  while (now_ms() < t_end) {
    int s = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
    if (s < 0) return false;
    if (connect(s, (sockaddr*)&a, al) != 0) {
      close(s);
      usleep(2000);
      continue;
    }
    char byte = 0;
    iovec io{&byte, 1};
    char ctrl[CMSG_SPACE(2 * sizeof(int))] = {};
    msghdr m = {};
    m.msg_iov = &io;
    m.msg_iovlen = 1;
    m.msg_control = ctrl;
    m.msg_controllen = sizeof ctrl;
    const ssize_t r = recvmsg(s, &m, 0);
    close(s);
    cmsghdr* cm = CMSG_FIRSTHDR(&m);
    if (r != 1 || !cm || cm->cmsg_type != SCM_RIGHTS || cm->cmsg_len != CMSG_LEN(2 * sizeof(int))) return false;
    memcpy(fds, CMSG_DATA(cm), 2 * sizeof(int));
    return true;
  }
  fprintf(stderr, "liblam: multicast: no owner on socket %s\n", name);
  return false;
}

}  // namespace

bool mc_supported(int dev, std::string* why) {
  const Drv& d = drv();
  if (!d.ok) { *why = "driver entry points for multicast not found"; return false; }
  CUdevice cd;
  int v = 0;
  if (d.dev_get(&cd, dev) != CUDA_SUCCESS || d.attr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cd) != CUDA_SUCCESS || !v) {
    *why = "device " + std::to_string(dev) + " does not support multicast objects (NVSwitch / fabric manager)";
    return false;
  }
  return true;
}

lam_status mc_alloc_members(McTeam& t, const std::vector<int>& local_devs, uint64_t bytes) {
  const Drv& d = drv();
  if (!d.ok) return LAM_ECUDA;
  size_t g1 = 0, g2 = 0;
  CUmulticastObjectProp mp = mc_prop((int)t.devices.size(), bytes);
  if (!cu_ok(d.mc_gran(&g1, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity")) return LAM_ECUDA;
  CUmemAllocationProp ap = member_prop(t.devices.front());
  if (!cu_ok(d.mem_gran(&g2, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity")) return LAM_ECUDA;
  const uint64_t g = std::max<uint64_t>(std::max<size_t>(g1, g2), 1);
  t.size = (bytes + g - 1) / g * g;
  for (int dev : local_devs) {
    CUmemAllocationProp p = member_prop(dev);
    CUmemGenericAllocationHandle h = 0;
    if (cudaSetDevice(dev) != cudaSuccess) return LAM_ECUDA;
    CUresult r = d.mem_create(&h, t.size, &p, 0);
    if (r == CUDA_ERROR_OUT_OF_MEMORY) return LAM_ENOMEM;
    if (!cu_ok(r, "cuMemCreate")) return LAM_ECUDA;
    t.mem[dev] = h;
    CUdeviceptr va = 0;
    if (!cu_ok(d.reserve(&va, t.size, g, 0, 0), "cuMemAddressReserve")) return LAM_ECUDA;
    if (!cu_ok(d.map(va, t.size, 0, h, 0), "cuMemMap(member)")) {
      d.addr_free(va, t.size);
      return LAM_ECUDA;
    }
    t.va[dev] = (uint8_t*)(uintptr_t)va;
    // the owner's member (node 0's slots) is readable by this process's other team GPUs too (node 0's
    // slot data mapped everywhere); every other member only locally
    std::vector<CUmemAccessDesc> acc;
    for (int other : local_devs)
      if (other == dev || dev == t.owner_dev) {
        CUmemAccessDesc a = {};
        a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        a.location.id = other;
        a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        acc.push_back(a);
      }
    if (!cu_ok(d.access(va, t.size, acc.data(), acc.size()), "cuMemSetAccess(member)")) return LAM_ECUDA;
    if (cudaMemset((void*)va, 0, t.size) != cudaSuccess) return LAM_ECUDA;   // pad bytes / flags zero
  }
  return LAM_OK;
}

lam_status mc_setup(McTeam& t, const std::vector<int>& local_devs, bool owner, int n_peer_procs, const char* sock) {
  const Drv& d = drv();
  if (!d.ok) return LAM_ECUDA;
  const uint64_t timeout_ms = 60000;
  if (owner) {
    CUmulticastObjectProp mp = mc_prop((int)t.devices.size(), t.size);
    if (!cu_ok(d.create(&t.mc, &mp), "cuMulticastCreate")) return LAM_ECUDA;
    if (n_peer_procs > 0) {
      // the multicast object, and the owner's member (node 0's slot data, mapped in every process)
      int fds[2] = {-1, -1};
      if (!cu_ok(d.exp(&fds[0], t.mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0), "cuMemExportToShareableHandle") ||
          !cu_ok(d.exp(&fds[1], t.mem.at(t.owner_dev), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
                 "cuMemExportToShareableHandle(member)")) {
        for (int f : fds)
          if (f >= 0) close(f);
        return LAM_EIPC;
      }
      const bool ok = serve_fd(sock, fds, n_peer_procs, timeout_ms);
      close(fds[0]);
      close(fds[1]);
      if (!ok) return LAM_EIPC;
    }
  } else {
    int fds[2] = {-1, -1};
    if (!fetch_fd(sock, timeout_ms, fds)) return LAM_EIPC;
    bool ok = cu_ok(d.imp(&t.mc, (void*)(uintptr_t)fds[0], CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
                    "cuMemImportFromShareableHandle");
    CUmemGenericAllocationHandle om = 0;
    ok = ok && cu_ok(d.imp(&om, (void*)(uintptr_t)fds[1], CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
                     "cuMemImportFromShareableHandle(member)");
    close(fds[0]);
    close(fds[1]);
    if (!ok) return LAM_EIPC;
    t.owner_imported = om;
    // map the owner's member here, readable by this process's GPUs (over NVLink)
    CUdeviceptr va = 0;
    if (!cu_ok(d.reserve(&va, t.size, 0, 0, 0), "cuMemAddressReserve(owner member)")) return LAM_ECUDA;
    if (!cu_ok(d.map(va, t.size, 0, om, 0), "cuMemMap(owner member)")) {
      d.addr_free(va, t.size);
      return LAM_ECUDA;
    }
    t.owner_va = (uint8_t*)(uintptr_t)va;
    std::vector<CUmemAccessDesc> acc(local_devs.size());
    for (size_t i = 0; i < local_devs.size(); ++i) {
      acc[i].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      acc[i].location.id = local_devs[i];
      acc[i].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    }
    if (!cu_ok(d.access(va, t.size, acc.data(), acc.size()), "cuMemSetAccess(owner member)")) return LAM_ECUDA;
  }
  for (int dev : local_devs) {
    CUdevice cd;
    if (!cu_ok(d.dev_get(&cd, dev), "cuDeviceGet") || !cu_ok(d.add(t.mc, cd), "cuMulticastAddDevice")) return LAM_ECUDA;
  }
  for (int dev : local_devs) {   // blocks until every team device (in every process) was added
    if (cudaSetDevice(dev) != cudaSuccess) return LAM_ECUDA;
    if (!cu_ok(d.bind(t.mc, 0, t.mem[dev], 0, t.size, 0), "cuMulticastBindMem")) return LAM_ECUDA;
    t.bound.push_back(dev);
  }
  if (owner) {
    if (cudaSetDevice(t.owner_dev) != cudaSuccess) return LAM_ECUDA;
    CUdeviceptr va = 0;
    if (!cu_ok(d.reserve(&va, t.size, 0, 0, 0), "cuMemAddressReserve(mc)")) return LAM_ECUDA;
    if (!cu_ok(d.map(va, t.size, 0, t.mc, 0), "cuMemMap(mc)")) {
      d.addr_free(va, t.size);
      return LAM_ECUDA;
    }
    t.mc_va = (uint8_t*)(uintptr_t)va;
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = t.owner_dev;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    if (!cu_ok(d.access(va, t.size, &acc, 1), "cuMemSetAccess(mc)")) return LAM_ECUDA;
  }
  return LAM_OK;
}

void mc_release(McTeam& t) {
  const Drv& d = drv();
  if (!d.ok) return;
  if (t.owner_va) {
    d.unmap((CUdeviceptr)(uintptr_t)t.owner_va, t.size);
    d.addr_free((CUdeviceptr)(uintptr_t)t.owner_va, t.size);
    t.owner_va = nullptr;
  }
  if (t.owner_imported) d.mem_release(t.owner_imported);
  t.owner_imported = 0;
  if (t.mc_va) {
    d.unmap((CUdeviceptr)(uintptr_t)t.mc_va, t.size);
    d.addr_free((CUdeviceptr)(uintptr_t)t.mc_va, t.size);
    t.mc_va = nullptr;
  }
  for (int dev : t.bound) {
    CUdevice cd;
    if (d.dev_get(&cd, dev) == CUDA_SUCCESS) d.unbind(t.mc, cd, 0, t.size);
  }
  t.bound.clear();
  for (auto& kv : t.va) {
    d.unmap((CUdeviceptr)(uintptr_t)kv.second, t.size);
    d.addr_free((CUdeviceptr)(uintptr_t)kv.second, t.size);
  }
  t.va.clear();
  for (auto& kv : t.mem) d.mem_release(kv.second);
  t.mem.clear();
  if (t.mc) d.mem_release(t.mc);
  t.mc = 0;
}

}  // namespace lam
