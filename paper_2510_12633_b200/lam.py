"""Thin ctypes binding of liblam.so (include/lam.h): same names, argument marshalling only.

Every step of the path runs in liblam's CUDA kernels; this module only converts Python values to
the C structs.  There is no CPU fallback: `load()` raises if liblam.so is missing, and liblam
returns LAM_ECUDA when no GPU is present.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblam.so")

LAM_MAX_RANKS, LAM_MAX_NODES, LAM_MAX_ROLLOUTS, LAM_MAX_DEVICES, LAM_MAX_SLOTS = 64, 32, 64, 16, 4
LAM_OK, LAM_ENOVERSION, LAM_IDLE = 0, 1, 2
LAM_EINVAL, LAM_ESTALE, LAM_ECUDA, LAM_ECHECKSUM, LAM_ENOMEM = -1, -2, -3, -4, -5
LAM_ESHUTDOWN, LAM_EBUSY, LAM_ETIMEOUT, LAM_EIPC = -6, -7, -8, -9
LAM_FSDP2_DIM0, LAM_FSDP1_FLAT = 0, 1
LAM_REPLICATE, LAM_SHARD_DIM0, LAM_SHARD_DIM1, LAM_VOCAB_DIM0, LAM_HEAD_DIM0 = 0, 1, 2, 3, 4
LAM_TILE_TRANSPOSE, LAM_TILE_ZERO = 0x100, 0xFFFFFFFF
LAM_HOP_KERNEL, LAM_HOP_COPY_ENGINE, LAM_HOP_MULTICAST, LAM_HOP_TREE = 0, 1, 2, 4


class lam_model_dims(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("hidden", "intermediate", "layers", "heads", "kv_heads",
                                          "head_dim", "vocab")]


class lam_node_desc(C.Structure):
    _fields_ = [("part_device", C.c_int32 * LAM_MAX_RANKS), ("host_memory", C.c_int32)]


class lam_rollout_desc(C.Structure):
    _fields_ = [("node", C.c_int32), ("device", C.c_int32)]


class lam_config(C.Structure):
    _fields_ = [("model", lam_model_dims), ("actor_layout", C.c_int32), ("fsdp_size", C.c_int32),
                ("actor_device", C.c_int32 * LAM_MAX_RANKS), ("n_relays", C.c_int32),
                ("relay", lam_node_desc * LAM_MAX_NODES), ("slots", C.c_int32), ("chunk_bytes", C.c_uint64),
                ("t_start_s", C.c_double), ("t_byte_s", C.c_double), ("n_rollouts", C.c_int32),
                ("rollout", lam_rollout_desc * LAM_MAX_ROLLOUTS), ("proc_rank", C.c_int32),
                ("n_procs", C.c_int32), ("proc_of_device", C.c_int32 * LAM_MAX_DEVICES),
                ("shm_name", C.c_char * 64), ("pack_ctas", C.c_int32), ("hop_ctas", C.c_int32),
                ("pull_ctas", C.c_int32), ("spin_timeout_s", C.c_double), ("hop_mode", C.c_int32),
                ("heartbeat_timeout_s", C.c_double), ("pack_sms", C.c_int32)]


class lam_shard(C.Structure):
    _fields_ = [("tensor_id", C.c_uint32), ("_pad", C.c_uint32), ("elem_offset", C.c_uint64),
                ("elem_count", C.c_uint64), ("ptr", C.c_void_p)]


class lam_part(C.Structure):
    _fields_ = [("tensor_id", C.c_uint32), ("rule", C.c_int32)]


class lam_dst(C.Structure):
    _fields_ = [("parts", C.POINTER(lam_part)), ("n_parts", C.c_int32), ("transpose", C.c_int32),
                ("dst", C.c_void_p), ("dst_row_pitch_bytes", C.c_int64)]


class lam_tp_layout(C.Structure):
    _fields_ = [("tp_size", C.c_int32), ("tp_rank", C.c_int32), ("dsts", C.POINTER(lam_dst)),
                ("n_dsts", C.c_int32)]


class lam_chunk_header(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("version", "idx", "n", "bytes", "s1", "s2", "_p0", "_p1")]


class lam_plan_info(C.Structure):
    _fields_ = [("image_bytes", C.c_uint64), ("chunk_bytes", C.c_uint64), ("total_chunks", C.c_uint64),
                ("snapshot_bytes", C.c_uint64), ("params", C.c_uint64), ("n_tensors", C.c_int32),
                ("n_nodes", C.c_int32)]


class lam_segment_info(C.Structure):
    _fields_ = [("tensor_id", C.c_uint32), ("rank", C.c_uint32), ("elem0", C.c_uint64), ("count", C.c_uint64),
                ("image_off", C.c_uint64)]


class lam_copy_tile_info(C.Structure):
    _fields_ = [("src_off", C.c_uint64), ("dst", C.c_uint64), ("src_pitch", C.c_uint32), ("dst_pitch", C.c_uint32),
                ("rows", C.c_uint32), ("row_bytes", C.c_uint32), ("src_rank", C.c_uint32), ("align", C.c_uint32)]


class lam_hop_tile_info(C.Structure):
    _fields_ = [("region_off", C.c_uint64), ("chunk", C.c_uint32), ("rank", C.c_uint32), ("bytes", C.c_uint32),
                ("source", C.c_uint32)]


class lam_stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("publishes", "publish_busy", "hops_launched", "versions_skipped",
                                          "pulls", "checksum_errors", "timeouts", "plan_cache_hits",
                                          "plan_cache_misses", "chain_rebuilds", "chain_resumes",
                                          "last_repair_ns", "kernel_launches", "publish_ns_total",
                                          "publish_ns_max")]


_LIB = None


def load() -> C.CDLL:
    """Load liblam.so (fails loudly if it was not built — there is no fallback path)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    P, V = C.POINTER, C.c_void_p
    sig = {
        "lam_init": (C.c_int32, [P(lam_config), P(V)]),
        "lam_export_ipc": (C.c_int32, [V, V, C.c_size_t, P(C.c_size_t)]),
        "lam_import_ipc": (C.c_int32, [V, C.c_int32, V, C.c_size_t]),
        "lam_connect": (C.c_int32, [V]),
        "lam_destroy": (None, [V]),
        "lam_strerror": (C.c_char_p, [C.c_int32]),
        "lam_publish": (C.c_int32, [V, C.c_uint64, C.c_int32, P(lam_shard), C.c_int32, V, V]),
        "lam_relay_step": (C.c_int32, [V, P(C.c_int32)]),
        "lam_pull": (C.c_int32, [V, C.c_int32, P(lam_tp_layout), V, P(C.c_uint64)]),
        "lam_latest": (C.c_int32, [V, C.c_int32, P(C.c_uint64)]),
        "lam_get_plan_info": (C.c_int32, [V, P(lam_plan_info)]),
        "lam_get_stats": (C.c_int32, [V, P(lam_stats)]),
        "lam_read_image": (C.c_int32, [V, C.c_int32, C.c_uint64, C.c_uint64, C.c_uint64, V]),
        "lam_read_headers": (C.c_int32, [V, C.c_int32, C.c_uint64, P(lam_chunk_header), C.c_uint64, C.c_uint64]),
        "lam_pull_bytes": (C.c_int32, [V, C.c_int32, P(lam_tp_layout), P(C.c_uint64), P(C.c_uint64)]),
        "lam_set_profiling": (C.c_int32, [V, C.c_int32]),
        "lam_kernel_times": (C.c_int32, [V, P(C.c_double), P(C.c_uint64)]),
        "lam_debug_region": (C.c_int32, [V, C.c_int32, C.c_uint64, C.c_int32, P(V)]),
        "lam_debug_replica": (C.c_int32, [V, C.c_int32, C.c_uint64, C.c_int32, P(V)]),
        "lam_model_n_tensors": (C.c_int32, [P(lam_model_dims)]),
        "lam_model_tensor": (C.c_int32, [P(lam_model_dims), C.c_int32, C.c_char_p, C.c_int32,
                                         P(C.c_int64), P(C.c_int32)]),
        "lam_vllm_layout": (C.c_int32, [P(lam_model_dims), C.c_int32, P(lam_dst), C.c_int32, P(lam_part),
                                        C.c_int32, C.c_char_p, C.c_int32, P(C.c_int64), P(C.c_int64)]),
        "lam_plan_segments": (C.c_int64, [P(lam_model_dims), C.c_int32, C.c_int32, C.c_uint64,
                                          P(lam_segment_info), C.c_int64]),
        "lam_plan_tree_tiles": (C.c_int64, [P(lam_model_dims), C.c_int32, C.c_int32, C.c_uint64, C.c_int32, C.c_int32,
                                            C.c_uint64, P(lam_hop_tile_info), C.c_int64]),
        "lam_plan_copy_tiles": (C.c_int64, [P(lam_model_dims), C.c_int32, C.c_int32, C.c_uint64, P(lam_tp_layout),
                                            P(lam_copy_tile_info), C.c_int64]),
        "lam_optimal_chunks": (C.c_int64, [C.c_int32, C.c_double, C.c_double, C.c_double, C.c_int64]),
        "lam_chain_latency": (C.c_double, [C.c_int32, C.c_int64, C.c_double, C.c_double, C.c_double]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    L.lam_config_size.restype, L.lam_config_size.argtypes = C.c_size_t, []
    if L.lam_config_size() != C.sizeof(lam_config):
        raise RuntimeError(f"{LIB_PATH} was built for sizeof(lam_config) = {L.lam_config_size()}, the binding has "
                           f"{C.sizeof(lam_config)}: stale build, run __graft_entry__.build()")
    _LIB = L
    return L


EXPORTED = ["lam_config_size", "lam_init", "lam_export_ipc", "lam_import_ipc", "lam_connect", "lam_destroy", "lam_strerror",
            "lam_publish", "lam_relay_step", "lam_pull", "lam_latest", "lam_get_plan_info", "lam_get_stats",
            "lam_read_image", "lam_read_headers", "lam_debug_region", "lam_debug_replica", "lam_set_profiling", "lam_kernel_times", "lam_pull_bytes", "lam_model_n_tensors", "lam_model_tensor", "lam_vllm_layout",
            "lam_plan_segments", "lam_plan_copy_tiles", "lam_plan_tree_tiles", "lam_optimal_chunks", "lam_chain_latency"]


class LamError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {load().lam_strerror(status).decode()} ({status})")


def _check(st: int, what: str, ok=(LAM_OK,)) -> int:
    if st not in ok:
        raise LamError(st, what)
    return st


# ------------------------------------------------------------------------------ model helpers
def dims(H, I, L, nh, nkv, hd, V) -> lam_model_dims:
    return lam_model_dims(H, I, L, nh, nkv, hd, V)


def model_tensors(d: lam_model_dims) -> list[tuple[str, tuple[int, ...]]]:
    L = load()
    n = L.lam_model_n_tensors(C.byref(d))
    _check(0 if n > 0 else LAM_EINVAL, "lam_model_n_tensors")
    out, name, shape, nd = [], C.create_string_buffer(128), (C.c_int64 * 2)(), C.c_int32()
    for i in range(n):
        _check(L.lam_model_tensor(C.byref(d), i, name, 128, shape, C.byref(nd)), "lam_model_tensor")
        out.append((name.value.decode(), (shape[0], shape[1]) if nd.value == 2 else (shape[0],)))
    return out


@dataclass
class VllmDst:
    name: str
    rows: int
    cols: int
    parts: list[tuple[int, int]]          # (tensor_id, rule)


def vllm_layout(d: lam_model_dims, tp: int) -> list[VllmDst]:
    L = load()
    n = L.lam_vllm_layout(C.byref(d), tp, None, 0, None, 0, None, 0, None, None)
    _check(0 if n > 0 else LAM_EINVAL, f"lam_vllm_layout(tp={tp})")
    dsts, parts = (lam_dst * n)(), (lam_part * (4 * n))()
    names = C.create_string_buffer(128 * n)
    rows, cols = (C.c_int64 * n)(), (C.c_int64 * n)()
    got = L.lam_vllm_layout(C.byref(d), tp, dsts, n, parts, 4 * n, names, 128, rows, cols)
    _check(0 if got == n else LAM_EINVAL, "lam_vllm_layout")
    out = []
    for i in range(n):
        nm = C.string_at(C.addressof(names) + 128 * i).decode()
        ps = [(dsts[i].parts[j].tensor_id, dsts[i].parts[j].rule) for j in range(dsts[i].n_parts)]
        out.append(VllmDst(nm, rows[i], cols[i], ps))
    return out


class TPLayout:
    """A rollout TP rank's destination buffers (keeps the ctypes arrays alive)."""

    def __init__(self, tp_size: int, tp_rank: int, dsts: list[tuple], transpose: bool = False):
        """dsts: list of (parts [(tensor_id, rule)], device pointer, row pitch bytes or 0[, transpose]);
        `transpose` is the default K-major flag of entries without their own."""
        self._parts = [(lam_part * len(d[0]))(*[lam_part(t, r) for t, r in d[0]]) for d in dsts]
        self._dsts = (lam_dst * max(1, len(dsts)))()
        for i, d in enumerate(dsts):
            p, ptr, pitch = d[:3]
            tr = d[3] if len(d) > 3 else transpose
            self._dsts[i] = lam_dst(C.cast(self._parts[i], C.POINTER(lam_part)), len(p), int(bool(tr)), ptr, pitch)
        self.c = lam_tp_layout(tp_size, tp_rank, C.cast(self._dsts, C.POINTER(lam_dst)), len(dsts))


# ------------------------------------------------------------------------------------ context
@dataclass
class Config:
    model: lam_model_dims
    fsdp_size: int = 1
    actor_devices: list[int] = field(default_factory=lambda: [0])
    relays: list[list[int]] = field(default_factory=list)      # per relay node: device per actor rank
    rollouts: list[tuple[int, int]] = field(default_factory=list)  # (node, device)
    actor_layout: int = LAM_FSDP2_DIM0
    slots: int = 2
    chunk_bytes: int = 0
    t_start_s: float = 0.0
    t_byte_s: float = 0.0
    proc_rank: int = 0
    n_procs: int = 1
    proc_of_device: dict[int, int] | None = None            # default: every used device -> proc 0
    shm_name: str = ""
    pack_ctas: int = 0
    hop_ctas: int = 0
    pull_ctas: int = 0
    spin_timeout_s: float = 0.0
    hop_mode: int = LAM_HOP_KERNEL
    heartbeat_timeout_s: float = 0.0
    pack_sms: int = 0                                            # > 0: pack confined to SMs 0..pack_sms-1
    host_relays: list[int] = field(default_factory=list)     # relay nodes (1-based) kept in host memory

    def to_c(self) -> lam_config:
        c = lam_config()
        c.model = self.model
        c.actor_layout, c.fsdp_size, c.n_relays, c.slots = (self.actor_layout, self.fsdp_size,
                                                            len(self.relays), self.slots)
        for r, d in enumerate(self.actor_devices):
            c.actor_device[r] = d
        for i, node in enumerate(self.relays):
            for r, d in enumerate(node):
                c.relay[i].part_device[r] = d
            c.relay[i].host_memory = int(i + 1 in self.host_relays)
        c.chunk_bytes, c.t_start_s, c.t_byte_s = self.chunk_bytes, self.t_start_s, self.t_byte_s
        c.n_rollouts = len(self.rollouts)
        for i, (node, dev) in enumerate(self.rollouts):
            c.rollout[i] = lam_rollout_desc(node, dev)
        c.proc_rank, c.n_procs = self.proc_rank, self.n_procs
        for d in range(LAM_MAX_DEVICES):
            c.proc_of_device[d] = -1
        pod = self.proc_of_device
        if pod is None:
            used = set(self.actor_devices) | {d for n in self.relays for d in n} | {d for _, d in self.rollouts}
            pod = {d: 0 for d in used}
        for d, p in pod.items():
            c.proc_of_device[d] = p
        c.shm_name = self.shm_name.encode()
        c.pack_ctas, c.hop_ctas, c.pull_ctas, c.spin_timeout_s = (self.pack_ctas, self.hop_ctas, self.pull_ctas,
                                                                  self.spin_timeout_s)
        c.hop_mode = self.hop_mode
        c.heartbeat_timeout_s = self.heartbeat_timeout_s
        c.pack_sms = self.pack_sms
        return c


class Context:
    def __init__(self, cfg: Config):
        self.L = load()
        self.cfg = cfg
        self._c = cfg.to_c()
        h = C.c_void_p()
        _check(self.L.lam_init(C.byref(self._c), C.byref(h)), "lam_init")
        self.h = h
        self._keep = []

    # -- multi-process plumbing (bytes move through torch.distributed in the caller)
    def export_ipc(self) -> bytes:
        n = C.c_size_t()
        _check(self.L.lam_export_ipc(self.h, None, 0, C.byref(n)), "lam_export_ipc")
        buf = C.create_string_buffer(n.value)
        _check(self.L.lam_export_ipc(self.h, buf, n.value, C.byref(n)), "lam_export_ipc")
        return buf.raw[:n.value]

    def import_ipc(self, proc: int, blob: bytes) -> None:
        _check(self.L.lam_import_ipc(self.h, proc, blob, len(blob)), "lam_import_ipc")

    def connect(self) -> None:
        _check(self.L.lam_connect(self.h), "lam_connect")

    # -- the path
    def publish(self, version: int, rank: int, shards: list[tuple[int, int, int, int]], actor_stream: int = 0,
                reads_done: int | None = None) -> int:
        """shards: (tensor_id, elem_offset, elem_count, device_ptr).  Returns LAM_OK or LAM_EBUSY."""
        arr = (lam_shard * max(1, len(shards)))()
        for i, (t, off, cnt, ptr) in enumerate(shards):
            arr[i] = lam_shard(t, 0, off, cnt, ptr)
        st = self.L.lam_publish(self.h, version, rank, arr, len(shards), actor_stream, reads_done)
        return _check(st, "lam_publish", ok=(LAM_OK, LAM_EBUSY))

    def relay_step(self) -> tuple[int, int]:
        n = C.c_int32()
        st = self.L.lam_relay_step(self.h, C.byref(n))
        _check(st, "lam_relay_step", ok=(LAM_OK, LAM_IDLE))
        return st, n.value

    def pull(self, rollout: int, layout: TPLayout, stream: int = 0) -> int:
        v = C.c_uint64()
        st = self.L.lam_pull(self.h, rollout, C.byref(layout.c), stream, C.byref(v))
        _check(st, "lam_pull", ok=(LAM_OK, LAM_ENOVERSION))
        return v.value

    def latest(self, node: int) -> int:
        v = C.c_uint64()
        _check(self.L.lam_latest(self.h, node, C.byref(v)), "lam_latest", ok=(LAM_OK, LAM_ENOVERSION))
        return v.value

    def pull_stream(self, rollout: int, layout: TPLayout, stream: int = 0, done_event: int | None = None,
                    min_version: int = 1) -> int:
        """lam_pull_stream: pull the first version >= min_version, chunk by chunk as it arrives.
        Returns the version (0 if none is complete or in flight); LAM_EBUSY raises."""
        f = self.L.lam_pull_stream
        f.restype = C.c_int32
        f.argtypes = [C.c_void_p, C.c_int32, C.POINTER(lam_tp_layout), C.c_void_p, C.c_void_p, C.c_uint64,
                      C.POINTER(C.c_uint64)]
        v = C.c_uint64()
        st = f(self.h, rollout, C.byref(layout.c), stream, done_event, min_version, C.byref(v))
        _check(st, "lam_pull_stream", ok=(LAM_OK, LAM_ENOVERSION))
        return v.value

    def subscribe(self, rollout: int, layout: TPLayout, done_event: int | None = None) -> None:
        """lam_subscribe: the next publish on the rollout's (actor) GPU also writes its TP=1 buffers."""
        f = self.L.lam_subscribe
        f.restype = C.c_int32
        f.argtypes = [C.c_void_p, C.c_int32, C.POINTER(lam_tp_layout), C.c_void_p]
        _check(f(self.h, rollout, C.byref(layout.c), done_event), "lam_subscribe")

    def pull_state(self, rollout: int) -> tuple[int, int]:
        """(version, state): state 1 = chunks still arriving, 0 = done, < 0 = failed."""
        f = self.L.lam_pull_state
        f.restype = C.c_int32
        f.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_uint64), C.POINTER(C.c_int32)]
        v, s = C.c_uint64(), C.c_int32()
        _check(f(self.h, rollout, C.byref(v), C.byref(s)), "lam_pull_state")
        return v.value, s.value

    def fail_node(self, node: int) -> None:
        """Declare relay `node` failed: O(1) chain rebuild, successors resume (lam_fail_node)."""
        f = self.L.lam_fail_node
        f.restype, f.argtypes = C.c_int32, [C.c_void_p, C.c_int32]
        _check(f(self.h, node), "lam_fail_node")

    def plan_info(self) -> lam_plan_info:
        p = lam_plan_info()
        _check(self.L.lam_get_plan_info(self.h, C.byref(p)), "lam_get_plan_info")
        return p

    def stats(self) -> dict:
        s = lam_stats()
        _check(self.L.lam_get_stats(self.h, C.byref(s)), "lam_get_stats")
        return {n: getattr(s, n) for n, _ in lam_stats._fields_}

    def read_image(self, node: int, version: int, offset: int, nbytes: int) -> np.ndarray:
        out = np.empty(nbytes, dtype=np.uint8)
        _check(self.L.lam_read_image(self.h, node, version, offset, nbytes, out.ctypes.data), "lam_read_image")
        return out

    def read_headers(self, node: int, version: int, first: int = 0, count: int | None = None) -> list[dict]:
        if count is None:
            count = self.plan_info().total_chunks - first
        arr = (lam_chunk_header * max(1, count))()
        _check(self.L.lam_read_headers(self.h, node, version, arr, first, count), "lam_read_headers")
        return [dict(version=h.version, idx=h.idx, n=h.n, bytes=h.bytes, s1=h.s1, s2=h.s2) for h in arr[:count]]

    def pull_bytes(self, rollout: int, layout: TPLayout) -> tuple[int, int]:
        """(local, remote) bytes a pull of `layout` reads (remote = over NVLink)."""
        a, b = C.c_uint64(), C.c_uint64()
        _check(self.L.lam_pull_bytes(self.h, rollout, C.byref(layout.c), C.byref(a), C.byref(b)), "lam_pull_bytes")
        return a.value, b.value

    def set_profiling(self, on: bool) -> None:
        _check(self.L.lam_set_profiling(self.h, int(on)), "lam_set_profiling")

    def set_pack_sms(self, sms: int) -> None:
        _check(self.L.lam_set_pack_sms(self.h, int(sms)), "lam_set_pack_sms")

    def kernel_times(self) -> dict:
        """{'pack'|'hop'|'pull': (total_ms, launches)} of completed launches since the last call."""
        ms, n = (C.c_double * 3)(), (C.c_uint64 * 3)()
        _check(self.L.lam_kernel_times(self.h, ms, n), "lam_kernel_times")
        return {k: (ms[i], n[i]) for i, k in enumerate(("pack", "hop", "pull"))}

    def debug_region(self, node: int, version: int, rank: int) -> int:
        p = C.c_void_p()
        _check(self.L.lam_debug_region(self.h, node, version, rank, C.byref(p)), "lam_debug_region")
        return p.value

    def debug_replica(self, device: int, version: int, rank: int) -> int:
        p = C.c_void_p()
        _check(self.L.lam_debug_replica(self.h, device, version, rank, C.byref(p)), "lam_debug_replica")
        return p.value

    def close(self) -> None:
        if self.h:
            self.L.lam_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def plan_segments(d: lam_model_dims, layout: int, N: int, C_bytes: int) -> list[tuple[int, int, int, int, int]]:
    """(tensor_id, rank, elem0, count, image_off) of the library's image plan (host-only)."""
    L = load()
    n = L.lam_plan_segments(C.byref(d), layout, N, C_bytes, None, 0)
    _check(0 if n >= 0 else int(n), "lam_plan_segments")
    arr = (lam_segment_info * max(1, n))()
    L.lam_plan_segments(C.byref(d), layout, N, C_bytes, arr, n)
    return [(a.tensor_id, a.rank, a.elem0, a.count, a.image_off) for a in arr[:n]]


def plan_copy_tiles(d: lam_model_dims, layout: int, N: int, C_bytes: int, tp: TPLayout) -> list[lam_copy_tile_info]:
    """The library's pull copy plan for a TP layout (host-only; dst pointers used as integers)."""
    L = load()
    n = L.lam_plan_copy_tiles(C.byref(d), layout, N, C_bytes, C.byref(tp.c), None, 0)
    _check(0 if n >= 0 else int(n), "lam_plan_copy_tiles")
    arr = (lam_copy_tile_info * max(1, n))()
    L.lam_plan_copy_tiles(C.byref(d), layout, N, C_bytes, C.byref(tp.c), arr, n)
    return list(arr[:n])


def plan_tree_tiles(d: lam_model_dims, layout: int, N: int, C_bytes: int, n_relays: int, node: int,
                    peer_mask: int) -> list[tuple[int, int, int, int, int]]:
    """LAM_HOP_TREE: (region_off, chunk, rank, bytes, source node) of the tiles relay `node` walks, in order."""
    L = load()
    n = L.lam_plan_tree_tiles(C.byref(d), layout, N, C_bytes, n_relays, node, peer_mask, None, 0)
    _check(0 if n >= 0 else int(n), "lam_plan_tree_tiles")
    arr = (lam_hop_tile_info * max(1, n))()
    L.lam_plan_tree_tiles(C.byref(d), layout, N, C_bytes, n_relays, node, peer_mask, arr, n)
    return [(a.region_off, a.chunk, a.rank, a.bytes, a.source) for a in arr[:n]]


def optimal_chunks(p: int, M: float, t_byte: float, t_start: float, k_cap: int = 1024) -> int:
    return load().lam_optimal_chunks(p, M, t_byte, t_start, k_cap)


def chain_latency(p: int, k: int, M: float, t_byte: float, t_start: float) -> float:
    return load().lam_chain_latency(p, k, M, t_byte, t_start)


class Ctl:
    """The control plane alone (lam_ctl_*; host-only, no GPU): the version-table state machine the
    runtime uses, on a POSIX shared-memory block shared by several processes (name != "")."""

    def __init__(self, name: str, create: bool, n_nodes: int, slots: int = 2, fsdp: int = 1,
                 hop_mode: int = LAM_HOP_KERNEL):
        L = self.L = load()
        P, V, I32, U64 = C.POINTER, C.c_void_p, C.c_int32, C.c_uint64
        for fn, res, args in [("lam_ctl_open", V, [C.c_char_p, I32, I32, I32, I32]),
                              ("lam_ctl_open_mode", V, [C.c_char_p, I32, I32, I32, I32, I32]), ("lam_ctl_close", None, [V]),
                              ("lam_ctl_publish", I32, [V, U64, I32, P(I32)]), ("lam_ctl_pack_done", I32, [V, I32, U64]),
                              ("lam_ctl_start", I32, [V, I32, P(U64), P(I32)]),
                              ("lam_ctl_part_done", I32, [V, I32, I32, U64, I32, I32]),
                              ("lam_ctl_pin", U64, [V, I32, P(I32)]), ("lam_ctl_unpin", None, [V, I32, I32]),
                              ("lam_ctl_latest", U64, [V, I32]), ("lam_ctl_busy", I32, [V]),
                              ("lam_ctl_fail", I32, [V, I32]), ("lam_ctl_pred", I32, [V, I32]),
                              ("lam_ctl_slot", I32, [V, I32, I32, P(U64), P(I32), P(I32)]),
                              ("lam_ctl_heartbeat", U64, [V, I32, I32, U64, C.c_double, P(U64)]),
                              ("lam_ctl_dead_procs", U64, [V])]:
            f = getattr(L, fn)
            f.restype, f.argtypes = res, args
        self.h = L.lam_ctl_open_mode(name.encode(), int(create), n_nodes, slots, fsdp, hop_mode)
        if not self.h:
            raise LamError(LAM_EIPC, "lam_ctl_open")

    def publish(self, v: int, rank: int = 0):
        s = C.c_int32(-1)
        st = self.L.lam_ctl_publish(self.h, v, rank, C.byref(s))
        return st, s.value

    def pack_done(self, slot: int, v: int) -> bool:
        return bool(self.L.lam_ctl_pack_done(self.h, slot, v))

    def start(self, node: int):
        v, st = C.c_uint64(), C.c_int32()
        s = self.L.lam_ctl_start(self.h, node, C.byref(v), C.byref(st))
        return s, v.value, bool(st.value)

    def part_done(self, node: int, slot: int, v: int, n_parts: int = 1, err: int = LAM_OK) -> bool:
        return bool(self.L.lam_ctl_part_done(self.h, node, slot, v, n_parts, err))

    def pin(self, node: int):
        s = C.c_int32(-1)
        v = self.L.lam_ctl_pin(self.h, node, C.byref(s))
        return v, s.value

    def unpin(self, node: int, slot: int) -> None:
        self.L.lam_ctl_unpin(self.h, node, slot)

    def latest(self, node: int) -> int:
        return self.L.lam_ctl_latest(self.h, node)

    def busy(self) -> bool:
        return bool(self.L.lam_ctl_busy(self.h))

    def fail(self, node: int) -> bool:
        return bool(self.L.lam_ctl_fail(self.h, node))

    def pred(self, node: int) -> int:
        return self.L.lam_ctl_pred(self.h, node)

    def slot(self, node: int, slot: int):
        v, st, rd = C.c_uint64(), C.c_int32(), C.c_int32()
        self.L.lam_ctl_slot(self.h, node, slot, C.byref(v), C.byref(st), C.byref(rd))
        return v.value, st.value, rd.value

    def heartbeat(self, proc: int, n_procs: int, now_ns: int, limit_s: float, node_procs: list[int]) -> int:
        """Stamp `proc`; fail relay nodes of processes silent > limit_s.  Returns the failed-node mask."""
        arr = (C.c_uint64 * max(1, len(node_procs)))(*node_procs)
        return self.L.lam_ctl_heartbeat(self.h, proc, n_procs, now_ns, limit_s, arr)

    def dead_procs(self) -> int:
        return self.L.lam_ctl_dead_procs(self.h)

    def close(self) -> None:
        if self.h:
            self.L.lam_ctl_close(self.h)
            self.h = None
