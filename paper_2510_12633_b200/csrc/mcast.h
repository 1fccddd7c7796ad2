// Multicast team of the LAM_HOP_MULTICAST broadcast (mcast.cpp).  Internal to liblam.
#pragma once
#include <stdint.h>

#include <algorithm>
#include <map>
#include <string>
#include <vector>

#include "../../include/lam.h"

namespace lam {

struct McTeam {
  bool on = false;
  std::vector<int> devices;              // team: the actor GPU + every relay GPU (sorted, distinct)
  int owner_dev = -1;                    // the actor GPU (its process creates the object and stores)
  uint64_t size = 0;                     // bytes of every member (granularity-aligned)
  uint64_t flags_off = 0, flag_stride = 0;   // member layout: S x slot data, then S x chunk flags
  unsigned long long mc = 0;             // CUmemGenericAllocationHandle of the multicast object
  uint8_t* mc_va = nullptr;              // multicast VA (owner process only)
  std::map<int, unsigned long long> mem; // local team devices: member allocation
  std::map<int, uint8_t*> va;            // local team devices: member VA
  std::vector<int> bound;                // local devices bound to the object
  uint8_t* owner_va = nullptr;           // peer processes: the owner's member (node 0's slots) mapped here
  unsigned long long owner_imported = 0; // ... and its imported handle
};

// Is the device able to join a multicast team (NVSwitch + fabric manager)?
bool mc_supported(int dev, std::string* why);
// Create, map and zero the members of this process's team devices (t.devices set; t.size := bytes
// rounded up to the multicast and allocation granularities).
lam_status mc_alloc_members(McTeam& t, const std::vector<int>& local_devs, uint64_t bytes);
// Create (owner) or import (others) the multicast object, add this process's team devices, bind the
// members; the owner also maps the multicast VA.  n_peer_procs = other processes owning team devices
// (owner side); `sock` = abstract unix socket name for handing the object's descriptor over.
lam_status mc_setup(McTeam& t, const std::vector<int>& local_devs, bool owner, int n_peer_procs, const char* sock);
void mc_release(McTeam& t);

}  // namespace lam
