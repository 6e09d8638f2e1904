// Coarsest-level solvers (hierarchy.py:123-178).
//
//  * pcg80: the reference's fixed-count Jacobi-PCG on K + eps*I
//    (_fixed_jacobi_pcg, hierarchy.py:139-162) as ONE persistent cooperative
//    kernel: the 80 dependent steps never return to the host, dot products
//    are reduced deterministically across the grid (fixed partial order),
//    and the search-direction update is folded into the next SpMV (p is
//    double-buffered and recomputed for neighbours on the fly) so each step
//    costs two grid barriers instead of three.
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
  double* partials;    // 2 * gridDim.x
  unsigned* bar;       // monotonic arrival counter (zeroed before launch)
  double eps;
  int steps;
};

// Grid-wide barrier for a co-resident (cooperative) grid: one release-add per
// block on a monotonic counter and an acquire spin; the L1 is invalidated by
// the acquire so data written by other blocks before the barrier is seen.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// Every block sums the grid partials in the same fixed order (lane-strided
// accumulation + fixed xor tree in warp 0): identical bits on all blocks.
__device__ __forceinline__ double grid_total(const double* partials, int nb, double* sh) {
  if (threadIdx.x < 32) {
    double s = 0.0;
    for (int b = threadIdx.x; b < nb; b += 32) s += __ldcg(partials + b);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) *sh = s;
  }
  __syncthreads();
  const double v = *sh;
  __syncthreads();
  return v;
}

__device__ __forceinline__ void block_partial(double v, double* out, double* sm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sm[warp] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double s = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) __stcg(out, s);
  }
}

constexpr int kPcgNodes = 128;                 // nodes per block pass
constexpr int kPcgThreads = 3 * kPcgNodes;     // one thread per (node, dk plane)

// The reference pcg80 (hierarchy.py:139-162) as one persistent kernel.  Its
// dot products are not bit-reproducible in the reference either (OpenBLAS
// ddot), so the SpMV here uses FMA and three independent row accumulators.
__global__ void __launch_bounds__(kPcgThreads) pcg80_kernel(Pcg80Args P) {
  __shared__ double sm[kPcgThreads / 32];
  __shared__ double tot;
  __shared__ double rowpart[2][kPcgNodes][3];
  const int64_t nn = P.g.nnodes();
  const int64_t nd = 3 * nn;
  const int NX = P.g.nx + 1, NY = P.g.ny + 1;
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int nb = gridDim.x;
  double* partA = P.partials;
  double* partB = P.partials + nb;
  unsigned epoch = 0;

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
  block_partial(loc, &partB[blockIdx.x], sm);
  grid_barrier(P.bar, ++epoch * nb);
  double rz = grid_total(partB, nb, &tot);
  double beta = 0.0;
  for (int s = 0; s < P.steps; ++s) {
    const double* pold = (s & 1) ? P.p1 : P.p0;
    double* pnew = (s & 1) ? P.p0 : P.p1;
    const bool hb = s > 0;
    // phase A (one thread per node, 3 rows): p_new = z + beta*p_old recomputed
    // for the 27 neighbours, q = K p_new + eps p_new, partial p.q
    // Three threads per node (one per neighbour plane dk), 128 nodes per block
    // pass: consecutive threads of a part take consecutive nodes, so the SoA
    // stencil loads are coalesced; the three partial row sums meet in shared
    // memory in a fixed order.
    loc = 0.0;
    const int part = threadIdx.x / kPcgNodes;
    const int lnode = threadIdx.x % kPcgNodes;
    for (int64_t base = int64_t(blockIdx.x) * kPcgNodes; base < nn; base += int64_t(gridDim.x) * kPcgNodes) {
      const int64_t node = base + lnode;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      if (node < nn) {
        const int i = int(node % NX), j = int((node / NX) % NY), k = int(node / (int64_t(NX) * NY));
        const int dk = part - 1;
        if (k + dk >= 0 && k + dk <= P.g.nz) {
#pragma unroll
          for (int q9 = 0; q9 < 9; ++q9) {
            const int di = q9 % 3 - 1, dj = q9 / 3 - 1;
            if (i + di < 0 || i + di > P.g.nx || j + dj < 0 || j + dj > P.g.ny) continue;
            const int slot = part * 9 + q9;
            const int64_t m = node + di + int64_t(NX) * (dj + int64_t(NY) * dk);
            const double* a = P.A + int64_t(slot) * 9 * nn + node;
            double pv[3];
#pragma unroll
            for (int c = 0; c < 3; ++c)
              pv[c] = hb ? fma(beta, pold[3 * m + c], P.z[3 * m + c]) : pold[3 * m + c];
            a0 = fma(__ldg(a + 0 * nn), pv[0], a0);
            a0 = fma(__ldg(a + 1 * nn), pv[1], a0);
            a0 = fma(__ldg(a + 2 * nn), pv[2], a0);
            a1 = fma(__ldg(a + 3 * nn), pv[0], a1);
            a1 = fma(__ldg(a + 4 * nn), pv[1], a1);
            a1 = fma(__ldg(a + 5 * nn), pv[2], a1);
            a2 = fma(__ldg(a + 6 * nn), pv[0], a2);
            a2 = fma(__ldg(a + 7 * nn), pv[1], a2);
            a2 = fma(__ldg(a + 8 * nn), pv[2], a2);
          }
        }
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
          const double pc = hb ? fma(beta, pold[d], P.z[d]) : pold[d];
          pnew[d] = pc;
          const double qv = fma(P.eps, pc, av[c]);
          P.q[d] = qv;
          loc = fma(pc, qv, loc);
        }
      }
      __syncthreads();
    }
    block_partial(loc, &partA[blockIdx.x], sm);
    grid_barrier(P.bar, ++epoch * nb);
    const double pq = grid_total(partA, nb, &tot);
    if (!(pq > 0.0) || !isfinite(pq)) break;
    const double a = rz / pq;
    // phase B: x += a p; r -= a q; z = dinv r; rz_new
    loc = 0.0;
    for (int64_t d = tid; d < nd; d += stride) {
      const double pv = pnew[d];
      P.x[d] = fma(a, pv, P.x[d]);
      const double rv = fma(-a, P.q[d], P.r[d]);
      P.r[d] = rv;
      const double zv = P.dinv[d] * rv;
      P.z[d] = zv;
      loc = fma(rv, zv, loc);
    }
    block_partial(loc, &partB[blockIdx.x], sm);
    grid_barrier(P.bar, ++epoch * nb);
    const double rzn = grid_total(partB, nb, &tot);
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
  int dev = 0, nsm = 0, per_sm = 0;
  SG_CUDA(cudaGetDevice(&dev));
  SG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  SG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcg80_kernel, kPcgThreads, 0));
  const int64_t want = (g.d.nnodes() + kPcgNodes - 1) / kPcgNodes;
  // one block per SM at most: the barrier cost grows with the participant count
  const int64_t cap = int64_t(nsm) * std::min(std::max(per_sm, 1), 1);
  nblocks = int(std::max<int64_t>(1, std::min(want, cap)));
  partials.alloc(size_t(2 * nblocks));
  bar.alloc(1);
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
  SG_CUDA(cudaMemsetAsync(bar.p, 0, sizeof(unsigned), s));
  void* args[] = {&a};
  SG_CUDA(cudaLaunchCooperativeKernel((void*)pcg80_kernel, dim3(nblocks), dim3(kPcgThreads), args,
                                      0, s));
  SG_CHECK_LAUNCH();
}

// ------------------------------------------------------------------ dense
// Unblocked right-looking Cholesky of an n x n SPD matrix (row-major, lower
// triangle used) by one 1024-thread CTA; returns info > 0 on a non-positive
// pivot like LAPACK dpotrf.
__global__ void __launch_bounds__(1024) chol_kernel(int n, double* L, int* info) {
  __shared__ double piv;
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    if (threadIdx.x == 0) {
      const double d = L[int64_t(j) * n + j];
      if (!(d > 0.0) || !isfinite(d)) {
        bad = j + 1;
      } else {
        piv = sqrt(d);
        L[int64_t(j) * n + j] = piv;
      }
    }
    __syncthreads();
    if (bad) break;
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) L[int64_t(i) * n + j] /= piv;
    __syncthreads();
    // trailing update of the lower triangle: L[i][k] -= L[i][j] * L[k][j], k <= i
    const int m = n - j - 1;
    const int64_t tri = int64_t(m) * (m + 1) / 2;
    for (int64_t t = threadIdx.x; t < tri; t += blockDim.x) {
      // map t -> (ii, kk) with kk <= ii
      int ii = int((sqrt(8.0 * double(t) + 1.0) - 1.0) * 0.5);
      while (int64_t(ii) * (ii + 1) / 2 > t) --ii;
      while (int64_t(ii + 1) * (ii + 2) / 2 <= t) ++ii;
      const int kk = int(t - int64_t(ii) * (ii + 1) / 2);
      const int i = j + 1 + ii, k = j + 1 + kk;
      L[int64_t(i) * n + k] -= L[int64_t(i) * n + j] * L[int64_t(k) * n + j];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *info = bad;
}

// Column c of inv(L): forward substitution, one thread per column.
__global__ void trinv_kernel(int n, const double* __restrict__ L, double* __restrict__ Y) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  for (int i = 0; i < n; ++i) Y[int64_t(i) * n + c] = 0.0;
  Y[int64_t(c) * n + c] = 1.0 / L[int64_t(c) * n + c];
  for (int i = c + 1; i < n; ++i) {
    double s = 0.0;
    for (int t = c; t < i; ++t) s += L[int64_t(i) * n + t] * Y[int64_t(t) * n + c];
    Y[int64_t(i) * n + c] = -s / L[int64_t(i) * n + i];
  }
}

// Ainv[i][k] = sum_{t >= max(i,k)} Y[t][i] * Y[t][k]
__global__ void ytY_kernel(int n, const double* __restrict__ Y, double* __restrict__ Ai) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= int64_t(n) * n) return;
  const int i = int(q / n), k = int(q % n);
  double s = 0.0;
  for (int t = i > k ? i : k; t < n; ++t) s += Y[int64_t(t) * n + i] * Y[int64_t(t) * n + k];
  Ai[q] = s;
}

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
  DBuf<double> L(static_cast<size_t>(n * n)), Y(static_cast<size_t>(n * n));
  SG_CUDA(cudaMemcpyAsync(L.p, dense_with_eps, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, s));
  DBuf<int> info(1);
  chol_kernel<<<1, 1024, 0, s>>>(int(n), L.p, info.p);
  SG_CHECK_LAUNCH();
  int h_info = 0;
  info.download(&h_info, 1, s);
  SG_CUDA(cudaStreamSynchronize(s));
  if (h_info) return false;  // LinAlgError -> pcg80 fallback (hierarchy.py:172-178)
  trinv_kernel<<<grid_blocks(n, 64), 64, 0, s>>>(int(n), L.p, Y.p);
  SG_CHECK_LAUNCH();
  Ainv.alloc(size_t(n * n));
  ytY_kernel<<<grid_blocks(n * n, 256), 256, 0, s>>>(int(n), Y.p, Ainv.p);
  SG_CHECK_LAUNCH();
  SG_CUDA(cudaStreamSynchronize(s));
  return true;
}

void DenseInverse::solve(const double* r, double* x, cudaStream_t s) {
  SG_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * 3 * grid->d.nnodes(), s));
  gemv_node_kernel<<<grid_blocks(n * 32, 256), 256, 0, s>>>(n, grid->free2dof.p, Ainv.p, r, x);
  SG_CHECK_LAUNCH();
}

}  // namespace sg
