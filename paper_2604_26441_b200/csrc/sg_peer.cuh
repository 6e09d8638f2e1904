// Device side of the slab transport's rank-ordered sum (sg_peer.cu), shared
// with the fused PCG kernels (sg_krylov.cu): a reduction kernel finishes its
// in-grid sum and the cross-rank sum in the same launch (one thread of one
// block talks to the peers' mailboxes; the other blocks wait at the grid
// barrier), with the slot layout and epochs of peer_sum_kernel, so fused and
// separate sums interleave in one solve and give identical bits.
#pragma once
#include <cstddef>

namespace sg {

constexpr int kPeerMaxRanks = 64;
constexpr int kPeerSumMax = 8;  // doubles per allreduce slot
enum { PEER_CH_HALO = 0, PEER_CH_SUM = 1, PEER_CH_GATHER = 2 };

struct PeerSumDev {  // kernel parameter (by value)
  char* base[kPeerMaxRanks];  // every rank's mailbox (this rank's own included)
  int me = 0, world = 1;
  size_t sum_off = 0, flags_off = 0;
  unsigned long long* ep = nullptr;  // this rank's device epochs [channel]
};

__device__ __forceinline__ unsigned long long peer_ld_acq(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void peer_st_rel(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Spin until a peer's flag reaches v.  A rank that died mid-exchange must not
// hang the device: after 60 s the kernel traps (sticky error on this rank).
__device__ __forceinline__ void peer_wait_geq(const unsigned long long* p, unsigned long long v) {
  if (peer_ld_acq(p) >= v) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (peer_ld_acq(p) < v) {
    __nanosleep(128);
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 60ull * 1000000000ull) __trap();
  }
}

// Rank-ordered sum of one double, by ONE thread: store this rank's value into
// every rank's slot, raise the flags, wait for every rank, sum slot 0..world-1
// in order (the bits of peer_sum_kernel with n = 1).
__device__ __forceinline__ double peer_sum1(const PeerSumDev& P, double v) {
  const unsigned long long e = P.ep[PEER_CH_SUM] + 1;
  const int par = int(e & 1);
  for (int r = 0; r < P.world; ++r)
    reinterpret_cast<double*>(P.base[r] + P.sum_off)[(size_t(par) * P.world + P.me) * kPeerSumMax] = v;
  __threadfence_system();
  for (int r = 0; r < P.world; ++r)
    peer_st_rel(reinterpret_cast<unsigned long long*>(P.base[r] + P.flags_off) + 2 * P.world + P.me, e);
  const unsigned long long* fl =
      reinterpret_cast<const unsigned long long*>(P.base[P.me] + P.flags_off) + 2 * P.world;
  for (int r = 0; r < P.world; ++r) peer_wait_geq(fl + r, e);
  const double* sl = reinterpret_cast<const double*>(P.base[P.me] + P.sum_off) + size_t(par) * P.world * kPeerSumMax;
  double acc = __ldcg(sl);
  for (int r = 1; r < P.world; ++r) acc += __ldcg(sl + size_t(r) * kPeerSumMax);
  P.ep[PEER_CH_SUM] = e;
  return acc;
}

struct PeerComm;
// the device view of a peer transport's sum channel (false: no peer transport)
bool peer_sum_dev(const PeerComm* p, PeerSumDev& out);

}  // namespace sg
