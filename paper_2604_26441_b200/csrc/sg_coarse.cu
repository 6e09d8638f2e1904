// Coarsest-level solvers (hierarchy.py:123-178).
//
//  * pcg80: the reference's fixed-count Jacobi-PCG on K + eps*I
//    (_fixed_jacobi_pcg, hierarchy.py:139-162) as ONE persistent cooperative
//    kernel (one block per SM): the 80 dependent steps never return to the
//    host.  The contiguous-range kernel below keeps its operator rows in
//    shared memory; per step: phase A (q = (K+eps I) p with p = z + beta
//    p_old recomputed for the neighbours on the fly, branch-free), a grid
//    all-reduce (counter barrier + every block summing the block partials in
//    index order: deterministic), phase B (x, r, z updates) and a second
//    all-reduce.  The default is the brick-partitioned pipelined kernel
//    (pcg80_brick_kernel<2>) further down, with its rows in tensor memory.
//  * dense: Cholesky of K + eps*I computed on device at setup, then the
//    explicit inverse, so each V-cycle's coarsest solve is one GEMV.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include "sg_coarse.cuh"

namespace sg {

struct Pcg80Args {
  GridDesc g;
  const double* A;     // stencil SoA (243 * nn)
  const double* dinv;  // 1/(diag+eps), 0 on fixed
  const double* b;
  double* x;
  double* r;
  double* z;
  double* p0;
  double* p1;
  double* q;
  double* partials;    // [2][gridDim.x] block partials (double-buffered by epoch parity)
  unsigned* bar;       // monotonic arrival counter
  double eps;
  int steps;
  int cache_slots;     // stencil slots resident in shared memory (single-pass grids)
  long long* trace;    // optional: %globaltimer stamps of every block, step 10 (8 per block)
};

#define PCG_STAMP(k)                                                                  \
  do {                                                                                \
    if (P.trace && s == 10 && threadIdx.x == 0) {                                     \
      long long t_;                                                                   \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                          \
      P.trace[blockIdx.x * 8 + k] = t_;                                               \
    }                                                                                 \
  } while (0)

constexpr int kPcgNodes = 128;                 // nodes per block pass
constexpr int kPcgThreads = 3 * kPcgNodes;     // one thread per (node, dk plane)

// Grid all-reduce: thread 0 of every block stores the block partial and
// arrives on a monotonic counter with a release reduction, then spins with
// acquire loads (one poller per block: polling every partial from every block
// contends on the same L2 lines and was measured 2.5x slower).  After the
// block barrier, threads 0..nb-1 load one partial each (a single L2 round
// trip) and the totals are summed in a fixed tree over the block index: every
// block obtains identical bits, independent of arrival order.
__device__ __forceinline__ void stamp(long long* tr, int k) {
  if (tr && threadIdx.x == 0) {
    long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    tr[blockIdx.x * 8 + k] = t_;
  }
}

// Development trace of the brick kernels: stamps k of steps 8..15 of every
// block, tr[(block * 8 + step - 8) * 8 + k].
__device__ __forceinline__ void stamp_s(long long* tr, int s, int k) {
  if (tr && s >= 8 && s < 16 && threadIdx.x == 0) {
    long long t_;
#ifdef SG_TRACE_CLOCK
    t_ = clock64();  // SM cycles: fine-grained within a block, not comparable across SMs
#else
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
#endif
    tr[(blockIdx.x * 8 + (s - 8)) * 8 + k] = t_;
  }
}

// Sum of the per-warp values sm[0..nw) by one warp in a fixed xor tree.
__device__ __forceinline__ double warp_sum_of(const double* sm, int nw, int lane) {
  double v = lane < nw ? sm[lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double grid_allreduce(double v, const Pcg80Args& P, unsigned epoch,
                                                 double* sm, long long* tr = nullptr) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = int((blockDim.x + 31) >> 5);
  if (lane == 0) sm[warp] = v;
  __syncthreads();
  const int nb = gridDim.x;
  double* part = P.partials + (epoch & 1) * nb;
  if (warp == 0) {
    const double s = warp_sum_of(sm, nw, lane);
    if (lane == 0) {
      __stcg(part + blockIdx.x, s);
      const unsigned target = epoch * unsigned(nb);
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(P.bar) : "memory");
      stamp(tr, 5);
      unsigned f;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(P.bar) : "memory");
      } while (f < target);
      stamp(tr, 6);
    }
  }
  __syncthreads();
  double t = int(threadIdx.x) < nb ? __ldcg(part + threadIdx.x) : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) sm[16 + warp] = t;
  __syncthreads();
  const double tot = warp_sum_of(sm + 16, nw, lane);
  stamp(tr, 7);
  return tot;
}

// The reference pcg80 (hierarchy.py:139-162).  Its dot products are not
// bit-reproducible in the reference either (OpenBLAS ddot), so the SpMV here
// uses FMA and independent row accumulators; reductions are deterministic.
__global__ void __launch_bounds__(kPcgThreads) pcg80_kernel(Pcg80Args P) {
  __shared__ double sm[32];  // [0,16): block partials, [16,32): partial sums
  __shared__ double rowpart[2][kPcgNodes][3];
  extern __shared__ double smA[];  // [cache_slots*9][kPcgNodes] operator rows of this block
  const int64_t nn = P.g.nnodes();
  const int64_t nd = 3 * nn;
  const int NX = P.g.nx + 1, NY = P.g.ny + 1;
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  unsigned epoch = 0;
  if (P.cache_slots > 0) {
    const int64_t n0 = int64_t(blockIdx.x) * kPcgNodes;
    const int total = P.cache_slots * 9 * kPcgNodes;
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
      const int t = idx / kPcgNodes, ln = idx % kPcgNodes;
      const int64_t node = n0 + ln;
      smA[idx] = node < nn ? __ldg(P.A + int64_t(t) * nn + node) : 0.0;
    }
    __syncthreads();
  }

  // x = 0; r = b; z = dinv*r; p = z; rz = r.z
  double loc = 0.0;
  for (int64_t d = tid; d < nd; d += stride) {
    const double rv = P.b[d];
    const double zv = P.dinv[d] * rv;
    P.x[d] = 0.0;
    P.r[d] = rv;
    P.z[d] = zv;
    P.p0[d] = zv;
    loc += rv * zv;
  }
  double rz = grid_allreduce(loc, P, ++epoch, sm);
  double beta = 0.0;
  const int part = threadIdx.x / kPcgNodes;  // neighbour plane dk = part - 1
  const int lnode = threadIdx.x % kPcgNodes;
  for (int s = 0; s < P.steps; ++s) {
    const double* pold = (s & 1) ? P.p1 : P.p0;
    double* pnew = (s & 1) ? P.p0 : P.p1;
    const bool hb = s > 0;
    PCG_STAMP(0);
    // phase A: q = (K + eps I) p_new, p_new = z + beta p_old
    loc = 0.0;
    for (int64_t base = int64_t(blockIdx.x) * kPcgNodes; base < nn; base += int64_t(gridDim.x) * kPcgNodes) {
      const int64_t node = base + lnode;
      const int64_t cn = node < nn ? node : nn - 1;
      const int i = int(cn % NX), j = int((cn / NX) % NY), k = int(cn / (int64_t(NX) * NY));
      const int kk = min(max(k + part - 1, 0), P.g.nz);
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      // branch-free: out-of-grid neighbours are clamped onto valid nodes;
      // their stencil entries are stored as exact zeros.
#pragma unroll
      for (int q9 = 0; q9 < 9; ++q9) {
        const int ii = min(max(i + q9 % 3 - 1, 0), P.g.nx);
        const int jj = min(max(j + q9 / 3 - 1, 0), P.g.ny);
        const int64_t m = ii + int64_t(NX) * (jj + int64_t(NY) * kk);
        const int slot = part * 9 + q9;
        const bool cached = slot < P.cache_slots;
        const double* a = cached ? smA + slot * 9 * kPcgNodes + lnode : P.A + int64_t(slot) * 9 * nn + cn;
        const int64_t st = cached ? kPcgNodes : nn;
        double pv[3];
#pragma unroll
        for (int c = 0; c < 3; ++c)
          // plain (L1-cacheable) loads: the barrier's acquire invalidated the
          // L1, and each neighbour value is reused by up to 27 rows of the block
          pv[c] = hb ? fma(beta, pold[3 * m + c], P.z[3 * m + c]) : pold[3 * m + c];
        a0 = fma(a[0 * st], pv[0], a0);
        a0 = fma(a[1 * st], pv[1], a0);
        a0 = fma(a[2 * st], pv[2], a0);
        a1 = fma(a[3 * st], pv[0], a1);
        a1 = fma(a[4 * st], pv[1], a1);
        a1 = fma(a[5 * st], pv[2], a1);
        a2 = fma(a[6 * st], pv[0], a2);
        a2 = fma(a[7 * st], pv[1], a2);
        a2 = fma(a[8 * st], pv[2], a2);
      }
      if (part > 0) {
        rowpart[part - 1][lnode][0] = a0;
        rowpart[part - 1][lnode][1] = a1;
        rowpart[part - 1][lnode][2] = a2;
      }
      __syncthreads();
      if (part == 0 && node < nn) {
        const double av[3] = {a0 + rowpart[0][lnode][0] + rowpart[1][lnode][0],
                              a1 + rowpart[0][lnode][1] + rowpart[1][lnode][1],
                              a2 + rowpart[0][lnode][2] + rowpart[1][lnode][2]};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int64_t d = 3 * node + c;
          const double pc = hb ? fma(beta, __ldcg(pold + d), __ldcg(P.z + d)) : __ldcg(pold + d);
          pnew[d] = pc;
          const double qv = fma(P.eps, pc, av[c]);
          P.q[d] = qv;
          loc = fma(pc, qv, loc);
        }
      }
      __syncthreads();
    }
    PCG_STAMP(1);
    const double pq = grid_allreduce(loc, P, ++epoch, sm, (P.trace && s == 10) ? P.trace : nullptr);
    PCG_STAMP(2);
    if (!(pq > 0.0) || !isfinite(pq)) break;
    const double a = rz / pq;
    // phase B: x += a p; r -= a q; z = dinv r; rz_new
    loc = 0.0;
    for (int64_t d = tid; d < nd; d += stride) {
      const double pv = __ldcg(pnew + d);
      P.x[d] = fma(a, pv, P.x[d]);
      const double rv = fma(-a, __ldcg(P.q + d), P.r[d]);
      P.r[d] = rv;
      const double zv = P.dinv[d] * rv;
      P.z[d] = zv;
      loc = fma(rv, zv, loc);
    }
    PCG_STAMP(3);
    const double rzn = grid_allreduce(loc, P, ++epoch, sm);
    PCG_STAMP(4);
    if (!(rzn > 0.0) || !isfinite(rzn)) break;
    beta = rzn / rz;
    rz = rzn;
  }
}

// ------------------------------------------------------------ brick pcg80
// Same algorithm, data-parallel over 3D node bricks (one brick per block,
// one block per SM) instead of contiguous node ranges:
//  * the operator rows stay on chip for all steps: variants 0/1 keep the
//    dj = -1 stencil row of each thread's dk plane in registers (27 doubles)
//    and the other 18 slots in shared memory (the full operator does not fit
//    in 227 KB); the pipelined variant 2 keeps 7 of its 9 rows in tensor
//    memory and 2 in shared memory (kBrTmRows);
//  * p lives in shared memory on the brick plus a one-node halo and is
//    updated there, p = z + beta p, for halo nodes too (the same expression
//    on the same bits as the owner's), so z is the only vector that crosses
//    blocks;
//  * z crosses blocks as 16-byte LL packets {lo, flag, hi, flag}: each 8-byte
//    half carries the writer's step flag, so a reader knows the value is
//    current without a memory fence (fences measured ~0.7 us each on B200);
//  * the owner thread of a node keeps x, r, D^-1, q of its node in registers;
//  * each grid all-reduce: block partial -> LL packet, relaxed arrival on a
//    64-bit counter, one poller, then warp 0 reads all packets (validated by
//    flag) and sums them in a fixed order: identical bits on every block.
//    Flags carry a launch sequence kept on device, so CUDA-graph replays never
//    accept a stale packet.
constexpr int kBrCap = 144;                  // max nodes per brick
constexpr int kBrThreads = 3 * kBrCap;       // one thread per (node, dk plane)
constexpr int kBrBlock = (kBrThreads + 31) / 32 * 32;  // full warps (shuffles, tcgen05 .aligned)
constexpr int kBrLn = kBrCap + (kBrBlock - kBrThreads);  // row pitch of the per-part partials
constexpr int kBrRegRows = 3;                // q9 = 0..2 (dj = -1) kept in registers
constexpr int kBrSmRows = 9 - kBrRegRows;
constexpr int kBrWinMax = 448;               // halo-window nodes
// pipelined variant: window rows stored at stride bx + 16 (row r of a warp's
// lanes then starts at bank residue r*bx mod 16, as if the rows were packed:
// the 64-bit window reads of a half-warp hit 16 distinct bank pairs), per
// component kBrWinS doubles; other variants / oversized windows: stride bx + 2
constexpr int kBrWinS = 1024;
constexpr int kBrFill = (3 * kBrWinMax + kBrBlock - 1) / kBrBlock;
constexpr int kBrOwnVec = 9 * kBrLn;        // pipelined variant: [part][comp][kBrLn] SpMV partials
constexpr int kBrStage = 2 * 160;            // pipelined variant: staged partial packets

struct BrickState {           // device-resident across launches (Pcg80::bstate)
  unsigned long long count;   // arrival counter (monotonic)
  unsigned long long origin;  // counter value when the next launch starts
  unsigned long long seq;     // launch sequence
};

struct BrickArgs {
  GridDesc g;
  const double* A;     // stencil SoA (243 * nn)
  const double* Apk;   // pipelined variants: operator packed per block (pcg80_pack_kernel)
  const double* dinv;  // node layout, 0 on fixed
  const double* b;     // node layout
  double* x;           // node layout
  uint4* zll;          // [3][nn] LL packets of z
  uint4* slots;        // [2][gridDim.x] LL packets of block partials
  BrickState* st;
  double eps;
  int steps;
  int sx, sy, sz;
  int nrep;            // variant 3: replicas of the partial-packet array (spread L2 polling)
  int poll_ns;         // variant 3: back-off between polling passes
  int winpad;          // variant 2: padded window rows (conflict-free half-warp reads)
  int recip;           // variant 2: beta, beta*gamma/alpha_prev from reciprocals formed
                       // during the halo wait (one division on the critical path, not three)
  long long* trace;
};

__device__ __forceinline__ void ll_store(uint4* a, double v, unsigned flag) {
  asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(a),
               "r"(unsigned(__double2loint(v))), "r"(flag), "r"(unsigned(__double2hiint(v))),
               "r"(flag) : "memory");
}
__device__ __forceinline__ uint4 ll_raw(const uint4* a) {
  uint4 v;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ bool ll_load(const uint4* a, unsigned flag, double& v) {
  unsigned lo, f0, hi, f1;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(lo), "=r"(f0), "=r"(hi), "=r"(f1) : "l"(a) : "memory");
  v = __hiloint2double(int(hi), int(lo));
  return f0 == flag && f1 == flag;
}

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double br_allreduce(double v, const BrickArgs& P, unsigned flag,
                                               unsigned long long target, double* red,
                                               double* tot) {
  v = wsum(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    const int nb = gridDim.x;
    uint4* sl = P.slots + (flag & 1) * nb;
    const double s = wsum(lane < int((blockDim.x + 31) >> 5) ? red[lane] : 0.0);
    if (lane == 0) {
      ll_store(sl + blockIdx.x, s, flag);
      asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(&P.st->count) : "memory");
      unsigned long long c;
      do {
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(c) : "l"(&P.st->count) : "memory");
      } while (c < target);
    }
    __syncwarp();
    double acc[5];
    bool ok;
    do {
      ok = true;
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const int bb = lane + 32 * k;
        acc[k] = 0.0;
        if (bb < nb) ok = ll_load(sl + bb, flag, acc[k]) && ok;
      }
    } while (!__all_sync(0xffffffffu, ok));
    const double t = wsum(acc[0] + acc[1] + acc[2] + acc[3] + acc[4]);
    if (lane == 0) *tot = t;
  }
  __syncthreads();
  return *tot;
}

// Two values in one all-reduce (the Chronopoulos-Gear step's (r.z, w.z)).
__device__ __forceinline__ void br_allreduce2(double v0, double v1, const BrickArgs& P,
                                              unsigned flag, unsigned long long target,
                                              double* red, double* tot, double& t0, double& t1) {
  v0 = wsum(v0);
  v1 = wsum(v1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    red[warp] = v0;
    red[16 + warp] = v1;
  }
  __syncthreads();
  if (warp == 0) {
    const int nb = gridDim.x;
    uint4* sl = P.slots + (flag & 1) * 2 * nb;
    const int nw = int((blockDim.x + 31) >> 5);
    const double s0 = wsum(lane < nw ? red[lane] : 0.0);
    const double s1 = wsum(lane < nw ? red[16 + lane] : 0.0);
    if (lane == 0) {
      ll_store(sl + blockIdx.x, s0, flag);
      ll_store(sl + nb + blockIdx.x, s1, flag);
      asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(&P.st->count) : "memory");
      unsigned long long c;
      do {
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(c) : "l"(&P.st->count) : "memory");
      } while (c < target);
    }
    __syncwarp();
    double a0[5], a1[5];
    bool ok;
    do {
      ok = true;
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const int bb = lane + 32 * k;
        a0[k] = 0.0;
        a1[k] = 0.0;
        if (bb < nb) {
          ok = ll_load(sl + bb, flag, a0[k]) && ok;
          ok = ll_load(sl + nb + bb, flag, a1[k]) && ok;
        }
      }
    } while (!__all_sync(0xffffffffu, ok));
    const double r0 = wsum(a0[0] + a0[1] + a0[2] + a0[3] + a0[4]);
    const double r1 = wsum(a1[0] + a1[1] + a1[2] + a1[3] + a1[4]);
    if (lane == 0) {
      tot[0] = r0;
      tot[1] = r1;
    }
  }
  __syncthreads();
  t0 = tot[0];
  t1 = tot[1];
}

// Split all-reduce of two values for the pipelined variant: publish the
// block partials and arrive (no wait), collect later (after the SpMV).
__device__ __forceinline__ void br_publish2(double v0, double v1, const BrickArgs& P,
                                            unsigned flag, double* red) {
  v0 = wsum(v0);
  v1 = wsum(v1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    red[warp] = v0;
    red[16 + warp] = v1;
  }
  __syncthreads();
  if (warp == 0) {
    const int nb = gridDim.x;
    // every replica [parity][r][2][nb] of the packet array (P.nrep >= 1)
    uint4* sl = P.slots + (flag & 1) * 2 * nb * P.nrep + lane * 2 * nb;
    const int nw = int((blockDim.x + 31) >> 5);
    const double s0 = wsum(lane < nw ? red[lane] : 0.0);
    const double s1 = wsum(lane < nw ? red[16 + lane] : 0.0);
    if (lane < P.nrep) {
      ll_store(sl + blockIdx.x, s0, flag);
      ll_store(sl + nb + blockIdx.x, s1, flag);
    }
  }
}
__device__ __forceinline__ void br_collect2(const BrickArgs& P, unsigned flag,
                                            unsigned long long target, double* tot, double& t0,
                                            double& t1) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    const int nb = gridDim.x;
    const uint4* sl = P.slots + (flag & 1) * 2 * nb;
    if (lane == 0) {
      unsigned long long c;
      do {
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(c) : "l"(&P.st->count) : "memory");
      } while (c < target);
    }
    __syncwarp();
    double a0[5], a1[5];
    bool ok;
    do {
      ok = true;
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const int bb = lane + 32 * k;
        a0[k] = 0.0;
        a1[k] = 0.0;
        if (bb < nb) {
          ok = ll_load(sl + bb, flag, a0[k]) && ok;
          ok = ll_load(sl + nb + bb, flag, a1[k]) && ok;
        }
      }
    } while (!__all_sync(0xffffffffu, ok));
    const double r0 = wsum(a0[0] + a0[1] + a0[2] + a0[3] + a0[4]);
    const double r1 = wsum(a1[0] + a1[1] + a1[2] + a1[3] + a1[4]);
    if (lane == 0) {
      tot[0] = r0;
      tot[1] = r1;
    }
  }
  __syncthreads();
  t0 = tot[0];
  t1 = tot[1];
}

// Tensor memory as a register-file extension (pipelined variant): the
// kBrRegRows operator rows a thread used to keep in registers live in its
// warp's TMEM lanes instead (warp w: lanes 32*(w%4).., columns 64*(w/4)..,
// one double = two 32-bit columns), read back one 9-entry row at a time with
// tcgen05.ld right before use.  That frees ~50 registers for the shared-memory
// load pipeline of the SpMV, which was latency-bound on register pressure.
constexpr int kBrTmRows = 7;     // q9 = 0..6 (63 doubles = 126 of a warp slot's 128 columns)
constexpr int kBrTmemCols = 512;  // 4 warp slots x 128 columns per lane quarter
constexpr int kMidQ = 4;  // SpMV row at which the partial packets are staged (2..4 best, 8: +2%)
__device__ __forceinline__ void tm_st18(uint32_t addr, const double (&v)[9]) {
  uint32_t r[18];
#pragma unroll
  for (int e = 0; e < 9; ++e) {
    r[2 * e] = unsigned(__double2loint(v[e]));
    r[2 * e + 1] = unsigned(__double2hiint(v[e]));
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};" ::"r"(addr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(addr + 16u), "r"(r[16]),
               "r"(r[17]) : "memory");
}
__device__ __forceinline__ void tm_ld18(uint32_t addr, double (&v)[9]) {
  uint32_t r[18];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(addr) : "memory");
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];"
               : "=r"(r[16]), "=r"(r[17]) : "r"(addr + 16u) : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int e = 0; e < 9; ++e) v[e] = __hiloint2double(int(r[2 * e + 1]), int(r[2 * e]));
}

// kVar = 2: pipelined Jacobi-PCG (Ghysels & Vanroose 2014, Alg. 4), the same
// iterates in exact arithmetic; the (r.u, w.u) all-reduce of a step is
// published before and collected after the step's SpMV n = A m, m = D^-1 w,
// so its latency hides behind the stencil work:
//   gamma = r.u, delta = w.u; m = D^-1 w; n = A m;
//   beta = gamma/gamma_prev; alpha = gamma/(delta - beta*gamma/alpha_prev);
//   z = n + beta z; q = m + beta q; s = w + beta s; p = u + beta p;
//   x += alpha p; r -= alpha s; u -= alpha q; w -= alpha z.
// m crosses blocks as LL packets in two parity buffers (a fast block writes
// step i+1 while a slow one may still read step i).
// kCG = false: the reference's Hestenes-Stiefel recurrence (two all-reduces
// per step).  kCG = true: the Chronopoulos-Gear form of the same Jacobi-PCG
// (identical iterates in exact arithmetic; one all-reduce of (r.z, w.z) per
// step with w = (K + eps I) z and s = A p carried by recurrence):
//   gamma = r.z, delta = w.z;  beta = gamma/gamma_prev;
//   p.Ap = delta - beta*gamma/alpha_prev;  alpha = gamma/p.Ap;
//   p = z + beta p; s = w + beta s; x += alpha p; r -= alpha s; z = D^-1 r.
// The reference's break tests map one to one: its rz_new test of step i-1 is
// the gamma test of step i, its p.q test the p.Ap test.
// shared-memory operator rows (doubles) and the whole dynamic allocation (bytes)
__host__ __device__ constexpr int br_smem_a(int var) {
  return 3 * (9 - (var >= 2 ? kBrTmRows : kBrRegRows)) * 9 * kBrCap;
}
__host__ __device__ constexpr int br_win_cs(int var) { return var == 2 ? kBrWinS : kBrWinMax; }
__host__ __device__ constexpr int br_smem_bytes(int var) {
  return int(sizeof(double)) * (br_smem_a(var) + 3 * br_win_cs(var) + kBrOwnVec) +
         int(sizeof(uint4)) * kBrStage +
         (var == 3 ? int(sizeof(double)) * (3 * kBrWinMax + 3 * kBrFill * kBrBlock) : 0);
}

// Operator of the pipelined variants packed per block at setup, in the order
// the kernel consumes it: the TMEM rows as [q/2][thread][2] (one coalesced
// 16-byte load per thread and row pair), then the shared-memory rows in the
// exact smA layout (one bulk async copy).
constexpr int kBrPkQ = (kBrTmRows * 9 + 1) / 2;        // double2 per thread
constexpr int kBrPkT = 2 * kBrPkQ * kBrBlock;           // doubles
constexpr int kBrPkS = 3 * (9 - kBrTmRows) * 9 * kBrCap;  // doubles
constexpr int kBrPk = kBrPkT + kBrPkS;                  // doubles per block
static_assert((kBrPkT * 8) % 16 == 0 && (kBrPkS * 8) % 16 == 0, "bulk copy alignment");

__global__ void __launch_bounds__(kBrBlock) pcg80_pack_kernel(BrickArgs P, double* out) {
  const int NX = P.g.nx + 1, NY = P.g.ny + 1, NZ = P.g.nz + 1;
  const int nn = NX * NY * NZ;
  const int bxi = int(blockIdx.x) % P.sx, byi = (int(blockIdx.x) / P.sx) % P.sy,
            bzi = int(blockIdx.x) / (P.sx * P.sy);
  const int x0 = bxi * NX / P.sx, y0 = byi * NY / P.sy, z0 = bzi * NZ / P.sz;
  const int bx = (bxi + 1) * NX / P.sx - x0, by = (byi + 1) * NY / P.sy - y0,
            bz = (bzi + 1) * NZ / P.sz - z0;
  const int nloc = bx * by * bz;
  const int t = threadIdx.x;
  const int part = min(t / kBrCap, 2), ln = t - part * kBrCap;
  const bool act = ln < nloc;
  const int lnc = act ? ln : 0;
  const int node = (x0 + lnc % bx) + NX * ((y0 + (lnc / bx) % by) + NY * (z0 + lnc / (bx * by)));
  double* o = out + int64_t(blockIdx.x) * kBrPk;
  for (int q = 0; q < 2 * kBrPkQ; ++q) {
    const double v = (q < kBrTmRows * 9 && act)
                         ? P.A[int64_t((part * 9 + q / 9) * 9 + q % 9) * nn + node] : 0.0;
    o[((q >> 1) * kBrBlock + t) * 2 + (q & 1)] = v;
  }
  constexpr int kSR = 9 - kBrTmRows;
  for (int idx = t; idx < kBrPkS; idx += blockDim.x) {
    const int e = idx / kBrCap, l = idx % kBrCap;
    const int pp = e / (kSR * 9), qq = (e / 9) % kSR, ent = e % 9;
    double v = 0.0;
    if (l < nloc) {
      const int gn = (x0 + l % bx) + NX * ((y0 + (l / bx) % by) + NY * (z0 + l / (bx * by)));
      v = P.A[int64_t((pp * 9 + kBrTmRows + qq) * 9 + ent) * nn + gn];
    }
    o[kBrPkT + idx] = v;
  }
}

// variant 3 adds a communication warp to the kBrBlock compute threads
__host__ __device__ constexpr int br_threads(int var) { return var == 3 ? kBrBlock + 32 : kBrBlock; }

template <int kVar>
__global__ void __launch_bounds__(br_threads(kVar), 1) pcg80_brick_kernel(BrickArgs P) {
  extern __shared__ double smdyn[];
  // register (TMEM for the pipelined variants) rows / shared-memory rows
  constexpr int kRR = kVar >= 2 ? kBrTmRows : kBrRegRows, kSR = 9 - kRR;
  double* smA = smdyn;             // [(part*kSR + row)*9 + entry][kBrCap]
  double* pw = smdyn + br_smem_a(kVar);  // [3][CS] p on the brick + halo
  constexpr int CS = br_win_cs(kVar);  // window doubles per component
  double* ov = pw + 3 * CS;  // [3][3][kBrLn] SpMV partials (pipelined variant)
  uint4* pst = reinterpret_cast<uint4*>(ov + kBrOwnVec);  // [2][160] staged packets
  __shared__ double rowpart[2][3][kBrLn];
  __shared__ double red[32];
  __shared__ double tot;
  __shared__ double tot2[2];
  const int NX = P.g.nx + 1, NY = P.g.ny + 1, NZ = P.g.nz + 1;
  const int nn = NX * NY * NZ;
  const int bxi = int(blockIdx.x) % P.sx, byi = (int(blockIdx.x) / P.sx) % P.sy,
            bzi = int(blockIdx.x) / (P.sx * P.sy);
  const int x0 = bxi * NX / P.sx, y0 = byi * NY / P.sy, z0 = bzi * NZ / P.sz;
  const int bx = (bxi + 1) * NX / P.sx - x0, by = (byi + 1) * NY / P.sy - y0,
            bz = (bzi + 1) * NZ / P.sz - z0;
  const int nloc = bx * by * bz;
  const int WX = bx + 2, WY = by + 2, WZ = bz + 2, wn = WX * WY * WZ;
  const int WXS = (kVar == 2 && P.winpad && (bx + 16) * WY * WZ <= CS) ? bx + 16 : WX;  // storage row stride
  const int t = threadIdx.x;
  // threads past 3*kBrCap (warp padding) are part 2 with ln >= kBrCap: never active
  const int part = min(t / kBrCap, 2), ln = t - part * kBrCap;
  const bool act = ln < nloc;
  const int lnc = act ? ln : 0;
  const int lx = lnc % bx, ly = (lnc / bx) % by, lz = lnc / (bx * by);
  const int node = (x0 + lx) + NX * ((y0 + ly) + NY * (z0 + lz));
  const bool owner = part == 0 && act;
  const int nb = gridDim.x;

  // launch sequence and counter origin (written by block 0 at the end of the
  // previous launch; every block reads them before its first arrival)
  const unsigned seq = unsigned(__ldcg(&P.st->seq));
  const unsigned long long c0 = __ldcg(&P.st->origin);
  const unsigned fbase = (seq + 1u) << 10;

  // operator rows: dj = -1 row of this thread's dk plane in registers (TMEM
  // for the pipelined variants), the rest in shared memory
  __shared__ uint32_t tm_base;
  __shared__ __align__(8) unsigned long long pk_bar;
  uint32_t tm_row = 0;  // this warp's TMEM address (lane quarter, column slot)
  if constexpr (kVar >= 2) {
    // packed operator: the shared-memory rows arrive by one bulk async copy
    // (mbarrier completion) while the threads stream their TMEM rows
    const double* blk = P.Apk + int64_t(blockIdx.x) * kBrPk;
    const unsigned bar_s = static_cast<unsigned>(__cvta_generic_to_shared(&pk_bar));
    if (t == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_s) : "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_s),
                   "n"(kBrPkS * 8) : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
          ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(smA))), "l"(blk + kBrPkT),
          "n"(kBrPkS * 8), "r"(bar_s) : "memory");
    }
    stamp_s(P.trace, 15, 0);
    const int warp = t >> 5;
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       static_cast<unsigned>(__cvta_generic_to_shared(&tm_base))),
                   "n"(kBrTmemCols) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    tm_row = tm_base + (uint32_t((warp & 3) * 32) << 16) + uint32_t((warp >> 2) * 128);
    // TMEM rows 0..3 then 4..6: 18 / 14 coalesced 16-byte loads in flight per thread
    const double2* src = reinterpret_cast<const double2*>(blk) + t;
    auto rows = [&](auto q0c, auto nrc) {
      constexpr int q0 = decltype(q0c)::value, nr = decltype(nrc)::value;
      constexpr int np = (nr * 9 + 1) / 2;
      double v[2 * np];
      // (threads past the brick's nodes hold zero padding: not loaded)
#pragma unroll
      for (int j = 0; j < np; ++j) {
        const double2 d = act ? __ldg(src + (q0 * 9 / 2 + j) * kBrBlock) : make_double2(0.0, 0.0);
        v[2 * j] = d.x;
        v[2 * j + 1] = d.y;
      }
#pragma unroll
      for (int q = 0; q < nr; ++q) {
        double r[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) r[e] = v[q * 9 + e];
        tm_st18(tm_row + uint32_t((q0 + q) * 18), r);
      }
    };
    stamp_s(P.trace, 15, 1);
    static_assert(kBrTmRows == 7, "row chunks below");
    if (warp < kBrBlock / 32) {  // (not the communication warp of variant 3)
      rows(std::integral_constant<int, 0>{}, std::integral_constant<int, 4>{});
      rows(std::integral_constant<int, 4>{}, std::integral_constant<int, 3>{});
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    stamp_s(P.trace, 15, 2);
    // shared-memory rows landed (phase 0 of the bulk-copy barrier)
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(bar_s) : "memory");
  }
  double areg[kRR * 9];  // variants 0/1 only
  if constexpr (kVar < 2) {
#pragma unroll
    for (int q = 0; q < kRR * 9; ++q)
      areg[q] = act ? __ldg(P.A + int64_t((part * 9 + q / 9) * 9 + q % 9) * nn + node) : 0.0;
  }
  for (int idx = t; kVar < 2 && idx < 3 * kSR * 9 * kBrCap; idx += blockDim.x) {
    const int e = idx / kBrCap, l = idx % kBrCap;
    const int pp = e / (kSR * 9), qq = (e / 9) % kSR, ent = e % 9;
    double v = 0.0;
    if (l < nloc) {
      const int gx = x0 + l % bx, gy = y0 + (l / bx) % by, gz = z0 + l / (bx * by);
      const int gn = gx + NX * (gy + NY * gz);
      v = __ldg(P.A + int64_t((pp * 9 + kRR + qq) * 9 + ent) * nn + gn);
    }
    smA[idx] = v;
  }
  // halo-window cells this thread stages each step (fixed for the launch)
  int fw[kBrFill], fg[kBrFill];
#pragma unroll
  for (int k = 0; k < kBrFill; ++k) {
    const int iw = t + k * kBrBlock;
    fw[k] = -1;
    fg[k] = -1;
    if (iw < 3 * wn) {
      const int c = iw / wn, w = iw - c * wn;
      const int wx = w % WX, wy = (w / WX) % WY, wz = w / (WX * WY);
      const int gx = x0 - 1 + wx, gy = y0 - 1 + wy, gz = z0 - 1 + wz;
      fw[k] = c * CS + (wz * WY + wy) * WXS + wx;
      if (gx >= 0 && gx < NX && gy >= 0 && gy < NY && gz >= 0 && gz < NZ)
        fg[k] = c * nn + gx + NX * (gy + NY * gz);
    }
  }

  const int wbase = ((lz + part) * WY + ly) * WXS + lx;
  const int wctr = ((lz + 1) * WY + ly + 1) * WXS + lx + 1;
  // stage the halo window of the LL vector written with flag zf; out-of-grid
  // cells are 0.  kAxpy: pw = beta*pw + v (p window), else pw = v.
  auto fill = [&](unsigned zf, bool axpy, double beta) {
    double zv[kBrFill];
    bool ok[kBrFill];
#pragma unroll
    for (int k = 0; k < kBrFill; ++k) {
      zv[k] = 0.0;
      ok[k] = fg[k] < 0 || ll_load(P.zll + fg[k], zf, zv[k]);
    }
    // not yet written (the neighbour is still finishing its step): re-poll
    // every pending cell together, one L2 round trip per pass
    bool all = true;
#pragma unroll
    for (int k = 0; k < kBrFill; ++k) all = all && ok[k];
    while (!all) {
      all = true;
#pragma unroll
      for (int k = 0; k < kBrFill; ++k) {
        if (!ok[k]) ok[k] = ll_load(P.zll + fg[k], zf, zv[k]);
        all = all && ok[k];
      }
    }
#pragma unroll
    for (int k = 0; k < kBrFill; ++k)
      if (fw[k] >= 0) pw[fw[k]] = axpy ? fma(beta, pw[fw[k]], zv[k]) : zv[k];
  };
  // y = K v on the window (the three dk planes summed by the owner thread)
  auto spmv_mid = [&](double av[3], auto&& mid) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
    for (int q9 = 0; q9 < 9; ++q9) {
      if (q9 == 6) mid();  // hook two thirds into the stencil work
      const int w = wbase + (q9 / 3) * WXS + q9 % 3;
      const double pv0 = pw[w], pv1 = pw[CS + w], pv2 = pw[2 * CS + w];
      double a[9];
#pragma unroll
      for (int e = 0; e < 9; ++e)
        a[e] = q9 < kRR ? areg[q9 * 9 + e]
                               : smA[((part * kSR + q9 - kRR) * 9 + e) * kBrCap + ln];
      a0 = fma(a[0], pv0, a0);
      a0 = fma(a[1], pv1, a0);
      a0 = fma(a[2], pv2, a0);
      a1 = fma(a[3], pv0, a1);
      a1 = fma(a[4], pv1, a1);
      a1 = fma(a[5], pv2, a1);
      a2 = fma(a[6], pv0, a2);
      a2 = fma(a[7], pv1, a2);
      a2 = fma(a[8], pv2, a2);
    }
    if (part > 0) {
      rowpart[part - 1][0][ln] = a0;
      rowpart[part - 1][1][ln] = a1;
      rowpart[part - 1][2][ln] = a2;
    }
    __syncthreads();
    av[0] = a0 + rowpart[0][0][ln] + rowpart[1][0][ln];
    av[1] = a1 + rowpart[0][1][ln] + rowpart[1][1][ln];
    av[2] = a2 + rowpart[0][2][ln] + rowpart[1][2][ln];
  };
  auto spmv = [&](double av[3]) { spmv_mid(av, [] {}); };

  if constexpr (kVar >= 2) {
    // Component ownership: thread (part, ln) owns component c = part of node
    // ln, so the ten per-DOF recurrences are scalars in every thread (no
    // 3-wide owner arrays: the registers go to the SpMV's load pipeline).
    const int nn3 = 3 * nn;  // one LL parity buffer
    const int c = part;
    double xr = 0.0, rr = 0.0, uu = 0.0, ww = 0.0, dv = 0.0;
    double zz = 0.0, qq = 0.0, ss = 0.0, pp = 0.0;
    double* rp3 = ov;  // [src part][comp][kBrLn] SpMV partials
    // full row sum of this thread's component: the three dk-plane partials
    // added in part order (p0 + p1) + p2 by every consumer
    // (two accumulators per row -- register rows / shared rows -- halve the
    // dependent DFMA chains)
    // compute-warp barrier (variant 3 has a communication warp outside it)
    auto csync = [&] {
      if constexpr (kVar == 3) asm volatile("bar.sync 3, %0;" ::"n"(kBrBlock) : "memory");
      else __syncthreads();
    };
    // mid() is called before stencil row qmid (the partial-packet staging hook)
    auto spmv_own_at = [&](auto qmid, auto&& mid) {
      double acc[2][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
#pragma unroll
      for (int q9 = 0; q9 < 9; ++q9) {
        if (q9 == decltype(qmid)::value) mid();
        const int w = wbase + (q9 / 3) * WXS + q9 % 3;
        const double pv0 = pw[w], pv1 = pw[CS + w], pv2 = pw[2 * CS + w];
        double a[9];
        if (q9 < kRR) {
          tm_ld18(tm_row + uint32_t(q9 * 18), a);
        } else {
#pragma unroll
          for (int e = 0; e < 9; ++e)
            a[e] = smA[((part * kSR + q9 - kRR) * 9 + e) * kBrCap + ln];
        }
        double* h = acc[q9 & 1];
        h[0] = fma(a[0], pv0, h[0]);
        h[0] = fma(a[1], pv1, h[0]);
        h[0] = fma(a[2], pv2, h[0]);
        h[1] = fma(a[3], pv0, h[1]);
        h[1] = fma(a[4], pv1, h[1]);
        h[1] = fma(a[5], pv2, h[1]);
        h[2] = fma(a[6], pv0, h[2]);
        h[2] = fma(a[7], pv1, h[2]);
        h[2] = fma(a[8], pv2, h[2]);
      }
      rp3[(part * 3 + 0) * kBrLn + ln] = acc[0][0] + acc[1][0];
      rp3[(part * 3 + 1) * kBrLn + ln] = acc[0][1] + acc[1][1];
      rp3[(part * 3 + 2) * kBrLn + ln] = acc[0][2] + acc[1][2];
      csync();
      return (rp3[c * kBrLn + ln] + rp3[(3 + c) * kBrLn + ln]) + rp3[(6 + c) * kBrLn + ln];
    };
    auto spmv_own = [&](auto&& mid) {
      return spmv_own_at(std::integral_constant<int, kMidQ>{}, mid);
    };
    auto tm_free = [&] {
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      if (t < 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm_base),
                     "n"(kBrTmemCols) : "memory");
    };
    // collect the (gamma, delta) partial packets of flag pf staged in pst
    // (re-polling stale ones), summed in a fixed order: identical on every block
    auto collect_staged = [&](unsigned pf, double& gam, double& del) {
      const uint4* sl = P.slots + (pf & 1) * 2 * nb;
      if (t < 32) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        double a0[5], a1[5];
        bool ok[10];
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const int bb = t + 32 * k;
          a0[k] = 0.0;
          a1[k] = 0.0;
          ok[2 * k] = ok[2 * k + 1] = true;
          if (bb < nb) {
            const uint4 v0 = pst[bb], v1 = pst[nb + bb];
            ok[2 * k] = v0.y == pf && v0.w == pf;
            ok[2 * k + 1] = v1.y == pf && v1.w == pf;
            a0[k] = __hiloint2double(int(v0.z), int(v0.x));
            a1[k] = __hiloint2double(int(v1.z), int(v1.x));
          }
        }
        bool all = true;
#pragma unroll
        for (int k = 0; k < 10; ++k) all = all && ok[k];
        while (!all) {
          uint4 v[10];
#pragma unroll
          for (int k = 0; k < 10; ++k)
            if (!ok[k]) v[k] = ll_raw(sl + (k & 1) * nb + t + 32 * (k >> 1));
          all = true;
#pragma unroll
          for (int k = 0; k < 10; ++k) {
            if (!ok[k]) {
              ok[k] = v[k].y == pf && v[k].w == pf;
              if (ok[k]) {
                const double d = __hiloint2double(int(v[k].z), int(v[k].x));
                if (k & 1) a1[k >> 1] = d; else a0[k >> 1] = d;
              }
            }
            all = all && ok[k];
          }
        }
        const double r0 = wsum(a0[0] + a0[1] + a0[2] + a0[3] + a0[4]);
        const double r1 = wsum(a1[0] + a1[1] + a1[2] + a1[3] + a1[4]);
        if (t == 0) {
          tot2[0] = r0;
          tot2[1] = r1;
        }
      }
      __syncthreads();
      gam = tot2[0];
      del = tot2[1];
    };
    auto stage_partials = [&](unsigned pf) {
      if (t < 32) {
        const uint4* sl = P.slots + (pf & 1) * 2 * nb;
        for (int q = t; q < 2 * nb; q += 32) {
          const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(pst + q));
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(sl + q) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      }
    };
    if constexpr (kVar == 3) {
      stamp_s(P.trace, 15, 3);
      // Early-halo pipelined CG with a communication warp.
      //  * Same recurrences as kVar = 2, but what crosses blocks is the raw
      //    SpMV result nv = A m of the brick, sent the moment the SpMV is done.
      //    Every block keeps the z and w recurrences for its whole halo window
      //    (fill cells) and forms the next m there itself,
      //    m' = D^-1 (w - alpha (fma(eps, m, nv) + beta z)), with the same
      //    expressions on the same bits as the owner, so the L2 round trip of
      //    the halo overlaps the all-reduce collect and the scalar update.
      //  * Warp kBrBlock/32 (the communication warp) owns the all-reduce: it
      //    forms and publishes the block partials, then polls every block's
      //    packets while the 14 compute warps run the next SpMV; the compute
      //    warps only wait on named barrier 2 for the result.
      //      barrier 1: compute warps arrive (per-warp partials in red[]),
      //                 comm warp syncs;
      //      barrier 2: comm warp arrives ((gamma, delta) in tot2), compute
      //                 warps sync;
      //      barrier 3: compute warps only (the SpMV partials, end of step).
      //  * Window m double-buffered; beta and gamma/alpha_prev use reciprocals
      //    formed after the fill (one division on the collect -> fill path).
      constexpr int kCompute = kBrBlock;
      const bool comm = t >= kCompute;
      double* pwA = pw;
      double* pwB = reinterpret_cast<double*>(pst + kBrStage);
      // fill cells: window index fw, LL index fg (halo) or rp3 index fo (own)
      // per fill cell recurrences in shared memory ([k][thread], conflict-free)
      int fo[kBrFill];
      double* fzh = pwB + 3 * kBrWinMax;
      double* fwh = fzh + kBrFill * kBrBlock;
      double* fdv = fwh + kBrFill * kBrBlock;
#define ZH(k) fzh[(k) * kBrBlock + t]
#define WH(k) fwh[(k) * kBrBlock + t]
#define DVH(k) fdv[(k) * kBrBlock + t]
      __shared__ int stop;
      if (t == 0) stop = 0;
#pragma unroll
      for (int k = 0; k < kBrFill; ++k) {
        fo[k] = -1;
        if (comm) continue;
        ZH(k) = 0.0;
        WH(k) = 0.0;
        DVH(k) = 0.0;
        const int iw = t + k * kBrBlock;
        if (iw < 3 * wn) {
          const int cc = iw / wn, w = iw - cc * wn;
          const int wx = w % WX, wy = (w / WX) % WY, wz = w / (WX * WY);
          if (wx >= 1 && wx <= bx && wy >= 1 && wy <= by && wz >= 1 && wz <= bz) {
            fo[k] = cc * kBrLn + (wx - 1) + bx * ((wy - 1) + by * (wz - 1));
          }
          double u0 = 0.0;
          if (fg[k] >= 0) {
            const int gnode = fg[k] - cc * nn;
            const double d = P.dinv[3 * gnode + cc];
            DVH(k) = d;
            u0 = d * P.b[3 * gnode + cc];
          }
          pwA[fw[k]] = u0;
          pwB[fw[k]] = 0.0;
          WH(k) = u0;  // holds u0 until the first fill turns it into w0
        }
      }
      if (act) {
        rr = P.b[3 * node + c];
        dv = P.dinv[3 * node + c];
        uu = dv * rr;
      }
      __syncthreads();
      stamp_s(P.trace, 15, 4);

      if (comm) {
        // ---------------------------------------------- communication warp
        const int lane = t - kCompute;
        constexpr int nw = kCompute / 32;
        unsigned epoch = 0;
        for (int s = 0; s < P.steps; ++s) {
          asm volatile("bar.sync 1, %0;" ::"n"(kCompute + 32) : "memory");
          if (stop) break;
          ++epoch;
          const unsigned pf = fbase | epoch;
          // replica r of the packet array: [parity][r][2][nb]; every block
          // writes all replicas, polls replica blockIdx % nrep
          uint4* sl0 = P.slots + (pf & 1) * 2 * nb * P.nrep;
          uint4* sl = sl0 + (int(blockIdx.x) % P.nrep) * 2 * nb;
          const double s0 = wsum(lane < nw ? red[lane] : 0.0);
          const double s1 = wsum(lane < nw ? red[16 + lane] : 0.0);
          if (lane < P.nrep) {
            ll_store(sl0 + lane * 2 * nb + blockIdx.x, s0, pf);
            ll_store(sl0 + lane * 2 * nb + nb + blockIdx.x, s1, pf);
          }
          // poll every block's packets (all loads of a pass in flight)
          double a0[5], a1[5];
          bool ok[10];
#pragma unroll
          for (int k = 0; k < 10; ++k) ok[k] = lane + 32 * (k >> 1) >= nb;
#pragma unroll
          for (int k = 0; k < 5; ++k) a0[k] = a1[k] = 0.0;
          bool all;
          do {
            uint4 v[10];
#pragma unroll
            for (int k = 0; k < 10; ++k)
              if (!ok[k]) v[k] = ll_raw(sl + (k & 1) * nb + lane + 32 * (k >> 1));
            all = true;
#pragma unroll
            for (int k = 0; k < 10; ++k) {
              if (!ok[k]) {
                ok[k] = v[k].y == pf && v[k].w == pf;
                if (ok[k]) {
                  const double d = __hiloint2double(int(v[k].z), int(v[k].x));
                  if (k & 1) a1[k >> 1] = d; else a0[k >> 1] = d;
                }
              }
              all = all && ok[k];
            }
            if (P.poll_ns && !all) __nanosleep(P.poll_ns);
          } while (!__all_sync(0xffffffffu, all));
          const double r0 = wsum(a0[0] + a0[1] + a0[2] + a0[3] + a0[4]);
          const double r1 = wsum(a1[0] + a1[1] + a1[2] + a1[3] + a1[4]);
          if (lane == 0) {
            tot2[0] = r0;
            tot2[1] = r1;
          }
          __syncwarp();
          asm volatile("bar.arrive 2, %0;" ::"n"(kCompute + 32) : "memory");
        }
      } else {
        // --------------------------------------------------- compute warps
        // w0 = A u0 + eps u0: no exchange needed (u0 is local data everywhere)
        double nv = spmv_own([] {});
        stamp_s(P.trace, 15, 5);
        if (act) {
          ww = fma(P.eps, uu, nv);
          ll_store(P.zll + c * nn + node, nv, fbase);
        }
        // per-warp partials of (gamma, delta) = (r.u, w.u) -> comm warp
        auto to_comm = [&](double lg, double ld) {
          lg = wsum(lg);
          ld = wsum(ld);
          if ((t & 31) == 0) {
            red[t >> 5] = lg;
            red[16 + (t >> 5)] = ld;
          }
          asm volatile("bar.arrive 1, %0;" ::"n"(kCompute + 32) : "memory");
        };
        to_comm(act ? rr * uu : 0.0, act ? ww * uu : 0.0);
        // halo cells: the LL loads are issued early (halo_issue, right after
        // the collect) and validated late (halo_finish), so their L2 round trip
        // overlaps the scalar update; own cells read the block's SpMV partials
        // from shared memory.  halo_issue only issues the loads: the flag test
        // -- the first use of the loaded registers -- is in halo_finish.
        uint4 zraw[kBrFill];
        auto halo_issue = [&](unsigned ph) {
          const uint4* base = P.zll + (ph & 1) * nn3;
#pragma unroll
          for (int k = 0; k < kBrFill; ++k) {
            zraw[k] = make_uint4(0u, 0u, 0u, 0u);
            if (fo[k] < 0 && fg[k] >= 0) zraw[k] = ll_raw(base + fg[k]);
          }
        };
        auto halo_finish = [&](unsigned ph, double* dst, auto&& upd) {
          const uint4* base = P.zll + (ph & 1) * nn3;
          const unsigned zf = fbase + ph;
          double zv[kBrFill];
          bool zok[kBrFill];
          bool all = true;
#pragma unroll
          for (int k = 0; k < kBrFill; ++k) {
            zok[k] = !(fo[k] < 0 && fg[k] >= 0) || (zraw[k].y == zf && zraw[k].w == zf);
            zv[k] = __hiloint2double(int(zraw[k].z), int(zraw[k].x));
            all = all && zok[k];
          }
          while (!all) {
            all = true;
#pragma unroll
            for (int k = 0; k < kBrFill; ++k) {
              if (!zok[k]) zok[k] = ll_load(base + fg[k], zf, zv[k]);
              all = all && zok[k];
            }
          }
#pragma unroll
          for (int k = 0; k < kBrFill; ++k) {
            if (fo[k] >= 0) {
              const int o = fo[k] % kBrLn, cc = fo[k] / kBrLn;
              zv[k] = (rp3[cc * kBrLn + o] + rp3[(3 + cc) * kBrLn + o]) + rp3[(6 + cc) * kBrLn + o];
            }
            if (fg[k] >= 0) dst[fw[k]] = upd(k, zv[k]);
          }
        };
        // window: w0 = fma(eps, u0, nv0), m0 = D^-1 w0
        halo_issue(0u);
        halo_finish(0u, pwB, [&](int k, double v) {
          const double w = fma(P.eps, WH(k), v);
          WH(k) = w;
          return DVH(k) * w;
        });
        csync();
        stamp_s(P.trace, 15, 6);
        double igprev = 0.0, iaprev = 0.0;
        for (int s = 0; s < P.steps; ++s) {
          double* cur = (s & 1) ? pwA : pwB;  // m_s
          double* nxt = (s & 1) ? pwB : pwA;  // m_{s+1}
          pw = cur;
          const int ts = s == 15 ? -1 : s;  // trace slot 15 holds the prologue stamps
          stamp_s(P.trace, ts, 0);
          nv = spmv_own([] {});
          if (act) ll_store(P.zll + ((s + 1) & 1) * nn3 + c * nn + node, nv, fbase + unsigned(s) + 1u);
          stamp_s(P.trace, ts, 3);
          asm volatile("bar.sync 2, %0;" ::"n"(kCompute + 32) : "memory");
          const double gam = tot2[0], del = tot2[1];
          stamp_s(P.trace, ts, 2);
          if (s + 1 < P.steps) halo_issue(unsigned(s) + 1u);
          double beta = 0.0, pap = del;
          bool brk = false;
          if (s > 0) {
            brk = !(gam > 0.0) || !isfinite(gam);
            beta = gam * igprev;
            pap = del - (beta * gam) * iaprev;
          }
          brk = brk || !(pap > 0.0) || !isfinite(pap);
          if (brk) {  // identical on every block; release the comm warp
            if (t == 0) stop = 1;
            csync();
            asm volatile("bar.arrive 1, %0;" ::"n"(kCompute + 32) : "memory");
            break;
          }
          const double al = gam / pap;
          stamp_s(P.trace, ts, 7);
          double lg = 0.0, ld = 0.0;
          if (act) {
            const double mv = cur[c * CS + wctr];
            const double n = fma(P.eps, mv, nv);
            zz = fma(beta, zz, n);
            qq = fma(beta, qq, mv);
            ss = fma(beta, ss, ww);
            pp = fma(beta, pp, uu);
            xr = fma(al, pp, xr);
            rr = fma(-al, ss, rr);
            uu = fma(-al, qq, uu);
            ww = fma(-al, zz, ww);
            lg = rr * uu;
            ld = ww * uu;
          }
          if (s + 1 == P.steps) break;
          to_comm(lg, ld);
          stamp_s(P.trace, ts, 1);
          halo_finish(unsigned(s) + 1u, nxt, [&](int k, double v) {
            const double n = fma(P.eps, cur[fw[k]], v);
            const double z = fma(beta, ZH(k), n);
            const double w = fma(-al, z, WH(k));
            ZH(k) = z;
            WH(k) = w;
            return DVH(k) * w;
          });
          stamp_s(P.trace, ts, 5);
          igprev = 1.0 / gam;
          iaprev = 1.0 / al;
          csync();
          stamp_s(P.trace, ts, 4);
        }
        if (act) P.x[3 * node + c] = xr;
        if (blockIdx.x == 0 && t == 0) {
          P.st->origin = c0;
          P.st->seq = seq + 1u;
        }
      }
      tm_free();
      return;
#undef ZH
#undef WH
#undef DVH
    }
    // phase 0: u0 = D^-1 b (flag fbase, buffer 0); w0 = A u0
    if (act) {
      rr = P.b[3 * node + c];
      dv = P.dinv[3 * node + c];
      uu = dv * rr;
      ll_store(P.zll + c * nn + node, uu, fbase);
    }
    auto fill_ph = [&](unsigned ph) {
      const uint4* base = P.zll + (ph & 1) * nn3;
      const unsigned zf = fbase + ph;
      double zv[kBrFill];
      bool ok[kBrFill];
#pragma unroll
      for (int k = 0; k < kBrFill; ++k) {
        zv[k] = 0.0;
        ok[k] = fg[k] < 0 || ll_load(base + fg[k], zf, zv[k]);
      }
      bool all = true;
#pragma unroll
      for (int k = 0; k < kBrFill; ++k) all = all && ok[k];
      while (!all) {
        all = true;
#pragma unroll
        for (int k = 0; k < kBrFill; ++k) {
          if (!ok[k]) ok[k] = ll_load(base + fg[k], zf, zv[k]);
          all = all && ok[k];
        }
      }
#pragma unroll
      for (int k = 0; k < kBrFill; ++k)
        if (fw[k] >= 0) pw[fw[k]] = zv[k];
    };
    fill_ph(0);
    __syncthreads();
    {
      const double av = spmv_own([] {});
      if (act) ww = fma(P.eps, uu, av);
    }
    unsigned epoch = 0;
    double gprev = 0.0, aprev = 0.0;
    double igprev = 0.0, iaprev = 0.0;  // 1/gamma_prev, 1/alpha_prev (formed off the critical path)
    for (int s = 0; s < P.steps; ++s) {
      stamp_s(P.trace, s, 0);
      // m = D^-1 w to the neighbours; (r.u, w.u) published
      double lg = 0.0, ld = 0.0;
      if (act) {
        ll_store(P.zll + ((s + 1) & 1) * nn3 + c * nn + node, dv * ww, fbase + unsigned(s) + 1u);
        lg = rr * uu;
        ld = ww * uu;
      }
      ++epoch;
      br_publish2(lg, ld, P, fbase | epoch, red);
      stamp_s(P.trace, s, 1);
      if (P.recip && s > 0) {  // the halo polls below wait anyway
        igprev = 1.0 / gprev;
        iaprev = 1.0 / aprev;
      }
      fill_ph(unsigned(s) + 1u);
      __syncthreads();
      stamp_s(P.trace, s, 5);
      // stage every block's partial packets into shared memory while the SpMV
      // runs (cp.async, L2 path); validated and re-polled afterwards
      const unsigned pf = fbase | epoch;
      const uint4* sl = P.slots + (pf & 1) * 2 * nb * P.nrep + (int(blockIdx.x) % P.nrep) * 2 * nb;
      // (issued two thirds into the SpMV, so late publishers are caught)
      const double nv = spmv_own([&] {
        if (t < 32) {
          for (int q = t; q < 2 * nb; q += 32) {
            const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(pst + q));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(sl + q) : "memory");
          }
          asm volatile("cp.async.commit_group;" ::: "memory");
        }
      });
      stamp_s(P.trace, s, 3);
      double gam, del;
      if (t < 32) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        double a0[5], a1[5];
        // staged copies first; every stale packet is then re-polled together
        // (all loads in flight at once: one L2 round trip per pass)
        bool ok[10];
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const int bb = t + 32 * k;
          a0[k] = 0.0;
          a1[k] = 0.0;
          ok[2 * k] = ok[2 * k + 1] = true;
          if (bb < nb) {
            const uint4 v0 = pst[bb], v1 = pst[nb + bb];
            ok[2 * k] = v0.y == pf && v0.w == pf;
            ok[2 * k + 1] = v1.y == pf && v1.w == pf;
            a0[k] = __hiloint2double(int(v0.z), int(v0.x));
            a1[k] = __hiloint2double(int(v1.z), int(v1.x));
          }
        }
        bool all = true;
#pragma unroll
        for (int k = 0; k < 10; ++k) all = all && ok[k];
        while (!all) {
          uint4 v[10];
#pragma unroll
          for (int k = 0; k < 10; ++k)
            if (!ok[k]) v[k] = ll_raw(sl + (k & 1) * nb + t + 32 * (k >> 1));
          all = true;
#pragma unroll
          for (int k = 0; k < 10; ++k) {
            if (!ok[k]) {
              ok[k] = v[k].y == pf && v[k].w == pf;
              if (ok[k]) {
                const double d = __hiloint2double(int(v[k].z), int(v[k].x));
                if (k & 1) a1[k >> 1] = d; else a0[k >> 1] = d;
              }
            }
            all = all && ok[k];
          }
        }
        stamp_s(P.trace, s, 6);
        const double r0 = wsum(a0[0] + a0[1] + a0[2] + a0[3] + a0[4]);
        const double r1 = wsum(a1[0] + a1[1] + a1[2] + a1[3] + a1[4]);
        if (t == 0) {
          tot2[0] = r0;
          tot2[1] = r1;
        }
      }
      __syncthreads();
      gam = tot2[0];
      del = tot2[1];
      stamp_s(P.trace, s, 2);
      double beta = 0.0, pap = del;
      if (s > 0) {
        if (!(gam > 0.0) || !isfinite(gam)) break;
        if (P.recip) {
          beta = gam * igprev;
          pap = del - (beta * gam) * iaprev;
        } else {
          beta = gam / gprev;
          pap = del - beta * gam / aprev;
        }
      }
      if (!(pap > 0.0) || !isfinite(pap)) break;
      const double al = gam / pap;
      if (act) {
        const double mv = pw[c * CS + wctr];
        const double n = fma(P.eps, mv, nv);
        zz = fma(beta, zz, n);
        qq = fma(beta, qq, mv);
        ss = fma(beta, ss, ww);
        pp = fma(beta, pp, uu);
        xr = fma(al, pp, xr);
        rr = fma(-al, ss, rr);
        uu = fma(-al, qq, uu);
        ww = fma(-al, zz, ww);
      }
      gprev = gam;
      aprev = al;
      stamp_s(P.trace, s, 4);
    }
    if (act) P.x[3 * node + c] = xr;
    if (blockIdx.x == 0 && t == 0) {
      P.st->origin = c0;  // this variant never arrives on the counter
      P.st->seq = seq + 1u;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (t < 32)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm_base),
                   "n"(kBrTmemCols) : "memory");
    return;
  }
  if constexpr (kVar == 1) {
    double xr[3] = {0.0, 0.0, 0.0}, rr[3] = {0.0, 0.0, 0.0}, dv[3] = {0.0, 0.0, 0.0};
    double pp[3] = {0.0, 0.0, 0.0}, ss[3] = {0.0, 0.0, 0.0};
    if (owner) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        rr[c] = P.b[3 * node + c];
        dv[c] = P.dinv[3 * node + c];
        ll_store(P.zll + c * nn + node, dv[c] * rr[c], fbase);
      }
    }
    unsigned epoch = 0;
    double gprev = 0.0, aprev = 0.0;
    for (int s = 0; s < P.steps; ++s) {
      if (P.trace && s == 10) stamp(P.trace, 0);
      fill(fbase + unsigned(s), false, 0.0);
      __syncthreads();
      if (P.trace && s == 10) stamp(P.trace, 5);
      double av[3];
      spmv(av);
      double lg = 0.0, ld = 0.0, zo[3] = {0.0, 0.0, 0.0}, wo[3] = {0.0, 0.0, 0.0};
      if (owner) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          zo[c] = pw[c * CS + wctr];
          wo[c] = fma(P.eps, zo[c], av[c]);
          lg = fma(rr[c], zo[c], lg);
          ld = fma(wo[c], zo[c], ld);
        }
      }
      if (P.trace && s == 10) stamp(P.trace, 1);
      ++epoch;
      double gam, del;
      br_allreduce2(lg, ld, P, fbase | epoch, c0 + epoch * nb, red, tot2, gam, del);
      if (P.trace && s == 10) stamp(P.trace, 2);
      double beta = 0.0, pap = del;
      if (s > 0) {
        if (!(gam > 0.0) || !isfinite(gam)) break;
        beta = gam / gprev;
        pap = del - beta * gam / aprev;
      }
      if (!(pap > 0.0) || !isfinite(pap)) break;
      const double al = gam / pap;
      if (owner) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          pp[c] = fma(beta, pp[c], zo[c]);
          ss[c] = fma(beta, ss[c], wo[c]);
          xr[c] = fma(al, pp[c], xr[c]);
          rr[c] = fma(-al, ss[c], rr[c]);
          if (s + 1 < P.steps) ll_store(P.zll + c * nn + node, dv[c] * rr[c], fbase + unsigned(s) + 1u);
        }
      }
      if (P.trace && s == 10) stamp(P.trace, 3);
      gprev = gam;
      aprev = al;
    }
    if (owner) {
#pragma unroll
      for (int c = 0; c < 3; ++c) P.x[3 * node + c] = xr[c];
    }
    if (blockIdx.x == 0 && t == 0) {
      P.st->origin = c0 + (unsigned long long)epoch * nb;
      P.st->seq = seq + 1u;
    }
    return;
  }

  // x = 0; r = b; z = dinv*r; p = z; rz = r.z
  double xr[3] = {0.0, 0.0, 0.0}, rr[3] = {0.0, 0.0, 0.0}, dv[3] = {0.0, 0.0, 0.0};
  double pown[3] = {0.0, 0.0, 0.0}, qown[3] = {0.0, 0.0, 0.0};
  double loc = 0.0;
  if (owner) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      rr[c] = P.b[3 * node + c];
      dv[c] = P.dinv[3 * node + c];
      const double zv = dv[c] * rr[c];
      ll_store(P.zll + c * nn + node, zv, fbase);
      loc = fma(rr[c], zv, loc);
    }
  }
  unsigned epoch = 0;
  ++epoch;
  double rz = br_allreduce(loc, P, fbase | epoch, c0 + epoch * nb, red, &tot);
  double beta = 0.0;
  for (int s = 0; s < P.steps; ++s) {
    if (P.trace && s == 10) stamp(P.trace, 0);
    // p = z + beta p on the brick + halo (z of step s carries flag fbase + s)
    fill(fbase + unsigned(s), s > 0, beta);
    __syncthreads();
    if (P.trace && s == 10) stamp(P.trace, 5);
    double av[3];
    spmv(av);
    loc = 0.0;
    if (owner) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        pown[c] = pw[c * CS + wctr];
        qown[c] = fma(P.eps, pown[c], av[c]);
        loc = fma(pown[c], qown[c], loc);
      }
    }
    if (P.trace && s == 10) stamp(P.trace, 1);
    ++epoch;
    const double pq = br_allreduce(loc, P, fbase | epoch, c0 + epoch * nb, red, &tot);
    if (P.trace && s == 10) stamp(P.trace, 2);
    if (!(pq > 0.0) || !isfinite(pq)) break;
    const double al = rz / pq;
    // x += a p; r -= a q; z = dinv r
    loc = 0.0;
    if (owner) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        xr[c] = fma(al, pown[c], xr[c]);
        rr[c] = fma(-al, qown[c], rr[c]);
        const double zv = dv[c] * rr[c];
        ll_store(P.zll + c * nn + node, zv, fbase + unsigned(s) + 1u);
        loc = fma(rr[c], zv, loc);
      }
    }
    if (P.trace && s == 10) stamp(P.trace, 3);
    ++epoch;
    const double rzn = br_allreduce(loc, P, fbase | epoch, c0 + epoch * nb, red, &tot);
    if (P.trace && s == 10) stamp(P.trace, 4);
    if (!(rzn > 0.0) || !isfinite(rzn)) break;
    beta = rzn / rz;
    rz = rzn;
  }
  if (owner) {
#pragma unroll
    for (int c = 0; c < 3; ++c) P.x[3 * node + c] = xr[c];
  }
  if (blockIdx.x == 0 && t == 0) {
    // every block arrived at all `epoch` all-reduces before block 0 left the last one
    P.st->origin = c0 + (unsigned long long)epoch * nb;
    P.st->seq = seq + 1u;
  }
}

// Brick split of the node grid for pcg80_brick_kernel: at most nsm bricks of
// at most kBrCap nodes, halo window <= kBrWinMax; smallest largest brick,
// then smallest window.  false = no such split (use the range kernel).
bool brick_plan(const GridDesc& g, int nsm, int& sx, int& sy, int& sz) {
  const int NX = g.nx + 1, NY = g.ny + 1, NZ = g.nz + 1;
  long best_b = 1L << 40, best_w = 1L << 40;
  bool found = false;
  for (int a = 1; a <= std::min(NX, nsm); ++a)
    for (int b = 1; a * b <= nsm && b <= NY; ++b)
      for (int c = 1; a * b * c <= nsm && c <= NZ; ++c) {
        const long ex = (NX + a - 1) / a, ey = (NY + b - 1) / b, ez = (NZ + c - 1) / c;
        const long vol = ex * ey * ez, win = (ex + 2) * (ey + 2) * (ez + 2);
        if (vol > kBrCap || win > kBrWinMax) continue;
        // ties: first found = fewest x splits = longest x extent (coalesced
        // halo fills; measured 454 us (3,7,7) vs 494 (7,3,7) vs 513 (7,7,3) at 26^3)
        if (vol < best_b || (vol == best_b && win < best_w)) {
          best_b = vol; best_w = win; sx = a; sy = b; sz = c; found = true;
        }
      }
  return found;
}

void Pcg80::setup(const Grid& g, const double* A, const double* diag, double eps_, int steps_,
                  cudaStream_t s) {
  grid = &g;
  Aptr = A;
  eps = eps_;
  steps = steps_;
  const int64_t nd = 3 * g.d.nnodes();
  dinv.alloc(size_t(nd));
  r.alloc(size_t(nd));
  z.alloc(size_t(nd));
  p0.alloc(size_t(nd));
  p1.alloc(size_t(nd));
  q.alloc(size_t(nd));
  std::vector<double> h(static_cast<size_t>(nd));
  SG_CUDA(cudaMemcpyAsync(h.data(), diag, sizeof(double) * nd, cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaStreamSynchronize(s));
  std::vector<uint8_t> fixed(static_cast<size_t>(nd), 1);
  std::vector<int32_t> f2d(static_cast<size_t>(g.n_free));
  SG_CUDA(cudaMemcpy(f2d.data(), g.free2dof.p, sizeof(int32_t) * g.n_free, cudaMemcpyDeviceToHost));
  for (int32_t d : f2d) fixed[size_t(d)] = 0;
  for (int64_t d = 0; d < nd; ++d) h[size_t(d)] = fixed[size_t(d)] ? 0.0 : 1.0 / (h[size_t(d)] + eps);
  dinv.upload(h.data(), h.size(), s);
  int dev = 0, nsm = 0, per_sm = 0, smem_optin = 0;
  SG_CUDA(cudaGetDevice(&dev));
  SG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  SG_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  // the brick kernels' packet flags carry the step in 10 bits (fbase = seq << 10):
  // longer fixed-step counts run on the contiguous-range kernel
  bool planned = !getenv("SG_PCG80_RANGE") && 2 * steps_ + 1 < 1024 &&
                 brick_plan(g.d, nsm, sx, sy, sz);
  if (planned && getenv("SG_BRICK")) {  // development override "sx,sy,sz"
    int a = 0, b = 0, c = 0;
    if (sscanf(getenv("SG_BRICK"), "%d,%d,%d", &a, &b, &c) == 3) { sx = a; sy = b; sz = c; }
  }
  if (planned) {
    brick = true;
    nblocks = sx * sy * sz;
    // 0: Hestenes-Stiefel (two all-reduces per step), 1: Chronopoulos-Gear,
    // 2: pipelined (the all-reduce hidden behind the SpMV; default), 3:
    // pipelined with the halo sent straight after the SpMV and a
    // communication warp for the all-reduce (measured slower: DESIGN 6b)
    variant = getenv("SG_PCG80_HS") ? 0 : getenv("SG_PCG80_CG") ? 1
            : getenv("SG_PCG80_EARLY") ? 3 : 2;
    constexpr int kBytes[4] = {br_smem_bytes(0), br_smem_bytes(1), br_smem_bytes(2),
                               br_smem_bytes(3)};
    smem_bytes = kBytes[variant];
    SG_REQUIRE(smem_bytes <= smem_optin, "pcg80 brick kernel shared memory");
    void* fns[4] = {(void*)pcg80_brick_kernel<0>, (void*)pcg80_brick_kernel<1>,
                    (void*)pcg80_brick_kernel<2>, (void*)pcg80_brick_kernel<3>};
    SG_CUDA(cudaFuncSetAttribute(fns[variant], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem_bytes));
    SG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fns[variant], br_threads(variant),
                                                          smem_bytes));
    SG_REQUIRE(per_sm >= 1, "pcg80 brick kernel cannot be resident");
    if (variant >= 2) {
      apk.alloc(size_t(nblocks) * kBrPk);
      BrickArgs a{};
      a.g = g.d;
      a.A = A;
      a.sx = sx;
      a.sy = sy;
      a.sz = sz;
      pcg80_pack_kernel<<<nblocks, kBrBlock, 0, s>>>(a, apk.p);
      SG_CHECK_LAUNCH();
    }
    nrep = 1;
    poll_ns = 0;
    if (variant >= 2) {
      if (getenv("SG_PCG80_NREP")) nrep = std::max(1, std::min(32, atoi(getenv("SG_PCG80_NREP"))));
      if (getenv("SG_PCG80_POLLNS")) poll_ns = std::max(0, atoi(getenv("SG_PCG80_POLLNS")));
    }
    slots.alloc(size_t(4 * nblocks * nrep));
    slots.zero(s);
    zll.alloc(size_t(6 * g.d.nnodes()));  // two LL parity buffers (pipelined variant)
    zll.zero(s);
    bstate.alloc(3);
    bstate.zero(s);
    SG_CUDA(cudaStreamSynchronize(s));
    return;
  }
  brick = false;
  const int64_t want = (g.d.nnodes() + kPcgNodes - 1) / kPcgNodes;
  // one block per SM: the barrier cost grows with the participant count, and a
  // single pass lets every block keep its operator rows in shared memory
  nblocks = int(std::max<int64_t>(1, std::min<int64_t>(want, nsm)));
  const int static_smem = 8 * 1024;
  const int per_slot = 9 * kPcgNodes * int(sizeof(double));
  cache_slots = 0;
  if (int64_t(nblocks) * kPcgNodes >= g.d.nnodes())
    cache_slots = std::max(0, std::min(27, (smem_optin - static_smem) / per_slot));
  smem_bytes = cache_slots * per_slot;
  SG_CUDA(cudaFuncSetAttribute(pcg80_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes));
  SG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcg80_kernel, kPcgThreads, smem_bytes));
  SG_REQUIRE(per_sm >= 1, "pcg80 kernel cannot be resident");
  partials.alloc(size_t(2 * nblocks));
  bar.alloc(32);
  SG_CUDA(cudaStreamSynchronize(s));
}

void Pcg80::solve(const double* b, double* x, cudaStream_t s) {
  if (brick) {
    BrickArgs a;
    a.g = grid->d;
    a.A = Aptr;
    a.Apk = apk.p;
    a.dinv = dinv.p;
    a.b = b;
    a.x = x;
    a.zll = zll.p;
    a.slots = slots.p;
    a.st = reinterpret_cast<BrickState*>(bstate.p);
    a.eps = eps;
    a.steps = steps;
    a.sx = sx;
    a.sy = sy;
    a.sz = sz;
    a.nrep = nrep;
    a.poll_ns = poll_ns;
    static const int recip = [] {  // SG_PCG80_RECIP=0: the three divisions (A/B)
      const char* e = std::getenv("SG_PCG80_RECIP");
      return e && e[0] == '0' ? 0 : 1;
    }();
    a.recip = recip;
    static const int winpad = [] {  // SG_PCG80_WINPAD=0: window rows at stride bx + 2 (A/B)
      const char* e = std::getenv("SG_PCG80_WINPAD");
      return e && e[0] == '0' ? 0 : 1;
    }();
    a.winpad = winpad;
    a.trace = trace;
    void* args[] = {&a};
    void* fn = variant == 3 ? (void*)pcg80_brick_kernel<3>
             : variant == 2 ? (void*)pcg80_brick_kernel<2>
             : variant == 1 ? (void*)pcg80_brick_kernel<1> : (void*)pcg80_brick_kernel<0>;
    SG_CUDA(cudaLaunchCooperativeKernel(fn, dim3(nblocks), dim3(br_threads(variant)),
                                        args, size_t(smem_bytes), s));
    SG_CHECK_LAUNCH();
    return;
  }
  Pcg80Args a;
  a.g = grid->d;
  a.A = Aptr;
  a.dinv = dinv.p;
  a.b = b;
  a.x = x;
  a.r = r.p;
  a.z = z.p;
  a.p0 = p0.p;
  a.p1 = p1.p;
  a.q = q.p;
  a.partials = partials.p;
  a.bar = bar.p;
  a.eps = eps;
  a.steps = steps;
  a.cache_slots = cache_slots;
  a.trace = trace;
  SG_CUDA(cudaMemsetAsync(bar.p, 0, sizeof(unsigned) * bar.n, s));
  void* args[] = {&a};
  SG_CUDA(cudaLaunchCooperativeKernel((void*)pcg80_kernel, dim3(nblocks), dim3(kPcgThreads), args,
                                      size_t(smem_bytes), s));
  SG_CHECK_LAUNCH();
}

// ------------------------------------------------------------------ dense
__global__ void gemv_node_kernel(int64_t nfree, const int32_t* __restrict__ f2d,
                                 const double* __restrict__ Ai, const double* __restrict__ r,
                                 double* __restrict__ x) {
  // one warp per output row: x[f2d[row]] = sum_c Ai[row][c] * r[f2d[c]]
  const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= nfree) return;
  const double* a = Ai + row * nfree;
  double s = 0.0;
  for (int64_t c = lane; c < nfree; c += 32) s += a[c] * r[f2d[c]];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) x[f2d[row]] = s;
}

bool DenseInverse::setup(const Grid& g, const double* dense_with_eps, cudaStream_t s) {
  grid = &g;
  n = g.n_free;
  SG_REQUIRE(n > 0 && n <= 20000, "dense coarsest size out of range");
  DBuf<double> L(static_cast<size_t>(n * n));
  SG_CUDA(cudaMemcpyAsync(L.p, dense_with_eps, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, s));
  Ainv.alloc(size_t(n * n));
  // blocked device Cholesky + inverse (sg_dense.cu); false = LinAlgError ->
  // pcg80 fallback (hierarchy.py:172-178)
  if (!dense_spd_inverse(int(n), L.p, Ainv.p, s)) {
    Ainv.release();
    return false;
  }
  return true;
}

void DenseInverse::solve(const double* r, double* x, cudaStream_t s) {
  SG_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * 3 * grid->d.nnodes(), s));
  gemv_node_kernel<<<grid_blocks(n * 32, 256), 256, 0, s>>>(n, grid->free2dof.p, Ainv.p, r, x);
  SG_CHECK_LAUNCH();
}

}  // namespace sg
