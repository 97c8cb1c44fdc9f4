// Peer-pointer plumbing shared by the fused data-parallel kernels.
#pragma once
#include <stdint.h>

namespace hm {

constexpr int kMaxPeers = 8;  // one NVLink/NVSwitch domain of a B200 box

// Passed by value as a kernel parameter: no device-side pointer table.
struct PeerPtrs {
  uint64_t p[kMaxPeers];
  int n;
};

// align: required alignment of every peer address (16 for page pools)
int make_peers(const uint64_t* ptrs, int n, PeerPtrs* out, unsigned align = 16);

}  // namespace hm
