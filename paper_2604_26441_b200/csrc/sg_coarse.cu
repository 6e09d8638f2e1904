// Coarsest-level solvers (hierarchy.py:123-178).
//
//  * pcg80: the reference's fixed-count Jacobi-PCG on K + eps*I
//    (_fixed_jacobi_pcg, hierarchy.py:139-162) as ONE persistent cooperative
//    kernel (one block per SM): the 80 dependent steps never return to the
//    host.  Each block keeps its operator rows resident in shared memory for
//    the whole solve; per step: phase A (q = (K+eps I) p with p = z + beta
//    p_old recomputed for the neighbours on the fly, branch-free), a grid
//    all-reduce (counter barrier + every block summing the block partials in
//    index order: deterministic), phase B (x, r, z updates) and a second
//    all-reduce.
//  * dense: Cholesky of K + eps*I computed on device at setup, then the
//    explicit inverse, so each V-cycle's coarsest solve is one GEMV.
#include <cmath>
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
  const int nw = int(blockDim.x >> 5);
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
