// 27-point 3x3-block stencil storage for the assembled (Galerkin) levels.
//
// Every Galerkin level of a structured trilinear hierarchy couples a node
// with its 3x3x3 neighbourhood, so the reference's CSR operators
// (hierarchy.py:262-265) are stored here without column indices as
// A[(slot*9 + ra*3 + cb) * n_nodes + node] (slot = (dk+1)*9 + (dj+1)*3 + (di+1)).
// Slot order equals ascending CSR column order, so the SpMV below sums each
// row in exactly the order scipy's csr_matvec does (FMA-free), and
// eliminated zeros are stored as 0.0 (adding them never changes a sum).
#include <numeric>
#include "sg_kernels.cuh"

namespace sg {

template <class T>
__device__ __forceinline__ T mul_rn(T a, T b);
template <>
__device__ __forceinline__ double mul_rn<double>(double a, double b) { return __dmul_rn(a, b); }
template <>
__device__ __forceinline__ float mul_rn<float>(float a, float b) { return __fmul_rn(a, b); }
template <class T>
__device__ __forceinline__ T add_rn(T a, T b);
template <>
__device__ __forceinline__ double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }
template <>
__device__ __forceinline__ float add_rn<float>(float a, float b) { return __fadd_rn(a, b); }

// Reads the TILED copy of the operator (stencil_tile: 32-node tiles, the 243
// coefficients of a tile contiguous), so each warp streams one contiguous
// 243 x 256 B block instead of 243 strided 256 B pieces (DRAM page locality).
// Branch-free and fully unrolled: out-of-grid neighbours are clamped onto the
// node itself, where the stored coefficients are exact zeros (the assembly
// zero-fills every slot), so all 243 coefficient loads and 81 neighbour loads
// of a row are independent and in flight together (the operator streams once
// per apply: memory-level parallelism is the bound).  The summation order is
// still the scipy csr_matvec order; a 0*x term only adds a signed zero.
template <class T>
__global__ void __launch_bounds__(128, 4) stencil_apply_kernel(GridDesc g, const T* __restrict__ At,
                                                            const T* __restrict__ x, T* __restrict__ y) {
  const int64_t nn = g.nnodes();
  const int64_t node = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (node >= nn) return;
  const int NX = g.nx + 1, NY = g.ny + 1;
  const int64_t NXY = int64_t(NX) * NY;
  // 32-bit index math (node < 2^31 for every level): 64-bit div/mod is a long
  // software sequence
  const int nd32 = int(node), jk = nd32 / NX;
  const int i = nd32 - jk * NX, j = jk % NY, k = jk / NY;
  const int64_t oi[3] = {i > 0 ? -1 : 0, 0, i < g.nx ? 1 : 0};
  const int64_t oj[3] = {j > 0 ? -NX : 0, 0, j < g.ny ? NX : 0};
  const int64_t ok[3] = {k > 0 ? -NXY : 0, 0, k < g.nz ? NXY : 0};
  T s0 = 0, s1 = 0, s2 = 0;
#pragma unroll
  for (int slot = 0; slot < 27; ++slot) {
    const int64_t nb = node + oi[slot % 3] + oj[(slot / 3) % 3] + ok[slot / 9];
    const T x0 = x[3 * nb], x1 = x[3 * nb + 1], x2 = x[3 * nb + 2];
    const T* a = At + (node >> 5) * (243 * 32) + slot * (9 * 32) + (node & 31);
    s0 = add_rn(s0, mul_rn(__ldcs(a + 0 * 32), x0));
    s0 = add_rn(s0, mul_rn(__ldcs(a + 1 * 32), x1));
    s0 = add_rn(s0, mul_rn(__ldcs(a + 2 * 32), x2));
    s1 = add_rn(s1, mul_rn(__ldcs(a + 3 * 32), x0));
    s1 = add_rn(s1, mul_rn(__ldcs(a + 4 * 32), x1));
    s1 = add_rn(s1, mul_rn(__ldcs(a + 5 * 32), x2));
    s2 = add_rn(s2, mul_rn(__ldcs(a + 6 * 32), x0));
    s2 = add_rn(s2, mul_rn(__ldcs(a + 7 * 32), x1));
    s2 = add_rn(s2, mul_rn(__ldcs(a + 8 * 32), x2));
  }
  y[3 * node] = s0;
  y[3 * node + 1] = s1;
  y[3 * node + 2] = s2;
}

// Fused epilogues for the FP64 Galerkin levels (smoothers.py:90-110 and the
// hierarchy.py:214 residual, same _rn operations as the elementwise kernels
// in sg_hier.cu, so the result is bit-identical to apply-then-update):
//   mode 1: r = b - Ax; d' = A*(dinv*r) [+ AC*d]; x' = x + d'  (x' != x)
//   mode 2: out = rr - Ax
__global__ void __launch_bounds__(128, 4) stencil_fused_kernel(GridDesc g, const double* __restrict__ At,
                                                            const double* __restrict__ x, int mode,
                                                            const double* __restrict__ b,
                                                            const double* __restrict__ dinv,
                                                            double* __restrict__ d, double* __restrict__ xout,
                                                            double A, double AC, int first) {
  const int64_t nn = g.nnodes();
  const int64_t node = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (node >= nn) return;
  const int NX = g.nx + 1, NY = g.ny + 1;
  const int64_t NXY = int64_t(NX) * NY;
  // 32-bit index math (node < 2^31 for every level): 64-bit div/mod is a long
  // software sequence
  const int nd32 = int(node), jk = nd32 / NX;
  const int i = nd32 - jk * NX, j = jk % NY, k = jk / NY;
  const int64_t oi[3] = {i > 0 ? -1 : 0, 0, i < g.nx ? 1 : 0};
  const int64_t oj[3] = {j > 0 ? -NX : 0, 0, j < g.ny ? NX : 0};
  const int64_t ok[3] = {k > 0 ? -NXY : 0, 0, k < g.nz ? NXY : 0};
  double s[3] = {0.0, 0.0, 0.0}, xc[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int slot = 0; slot < 27; ++slot) {
    const int64_t nb = node + oi[slot % 3] + oj[(slot / 3) % 3] + ok[slot / 9];
    const double x0 = x[3 * nb], x1 = x[3 * nb + 1], x2 = x[3 * nb + 2];
    if (slot == 13) {
      xc[0] = x0;
      xc[1] = x1;
      xc[2] = x2;
    }
    const double* a = At + (node >> 5) * (243 * 32) + slot * (9 * 32) + (node & 31);
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      s[r] = __dadd_rn(s[r], __dmul_rn(__ldcs(a + (3 * r + 0) * 32), x0));
      s[r] = __dadd_rn(s[r], __dmul_rn(__ldcs(a + (3 * r + 1) * 32), x1));
      s[r] = __dadd_rn(s[r], __dmul_rn(__ldcs(a + (3 * r + 2) * 32), x2));
    }
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int64_t q = 3 * node + r;
    if (mode == 2) {
      xout[q] = __dsub_rn(b[q], s[r]);
    } else {
      const double rv = __dsub_rn(b[q], s[r]);
      double dv = __dmul_rn(A, __dmul_rn(dinv[q], rv));
      if (!first) dv = __dadd_rn(dv, __dmul_rn(AC, d[q]));
      d[q] = dv;
      xout[q] = __dadd_rn(xc[r], dv);
    }
  }
}

// ---------------------------------------------------------------------------
// Symmetric ("upper") copy of an FP64 Galerkin stencil: only the diagonal
// slot 13 and the 13 lexicographically later slots 14..26 are stored (126
// of 243 coefficients per node, tiled like stencil_tile); a row's lower
// slot s < 13 uses the transpose of the block node j = i + off(s) stores in
// its mirror slot 26 - s.  The Galerkin operators are symmetric to rounding
// (P^T K P, K symmetric; the reference's assembled bits differ from exact
// symmetry by ~1 ulp), so y agrees with the full-stencil SpMV to ~1e-16
// relative while the operator streams 1008 instead of 1944 bytes per node
// from HBM -- the L1 smoother passes are HBM-bound at 92% of the roofline.
// Every row still sums its 27 blocks in the ascending-column (csr_matvec)
// order; deterministic.
constexpr int kSymQ = 126;
__global__ void stencil_sym_tile_kernel(int64_t nn, int64_t ntiles, const double* __restrict__ A,
                                        double* __restrict__ Ts) {
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= ntiles * kSymQ * 32) return;
  const int64_t lane = idx & 31, q = (idx >> 5) % kSymQ, tile = (idx >> 5) / kSymQ;
  const int64_t node = tile * 32 + lane;
  Ts[idx] = node < nn ? A[(13 * 9 + q) * nn + node] : 0.0;
}
void stencil_sym_tile(const Grid& g, const double* A, DBuf<double>& Ts, cudaStream_t s) {
  const int64_t nn = g.d.nnodes(), nt = (nn + 31) / 32;
  Ts.alloc(size_t(nt * kSymQ * 32));
  stencil_sym_tile_kernel<<<grid_blocks(nt * kSymQ * 32, 256), 256, 0, s>>>(nn, nt, A, Ts.p);
  SG_CHECK_LAUNCH();
}

// mode 0: y = A x; mode 1: Chebyshev step (stencil_fused_kernel mode 1);
// mode 2: out = rr - A x.  Same epilogue operations as the full-stencil kernels.
// Launch bounds (128, 4): 128 registers per thread, four blocks per SM -- more
// loads in flight per thread and fewer blocks streaming at once, so the
// neighbours' mirror blocks are still in L2 when read (DRAM 183 -> 144 MB per
// pass vs 140 MB algorithmic; 39.6 -> 31.9 us at 100^3; 3/5/6 blocks: 32.9 /
// 34.8 / 39.6 us).
__global__ void __launch_bounds__(128, 4) stencil_sym_kernel(GridDesc g, const double* __restrict__ Ts,
                                                          const double* __restrict__ x, int mode,
                                                          const double* __restrict__ b,
                                                          const double* __restrict__ dinv,
                                                          double* __restrict__ d, double* __restrict__ xout,
                                                          double A, double AC, int first) {
  const int64_t nn = g.nnodes();
  const int64_t node = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (node >= nn) return;
  const int NX = g.nx + 1, NY = g.ny + 1;
  const int64_t NXY = int64_t(NX) * NY;
  const int nd32 = int(node), jk = nd32 / NX;
  const int i = nd32 - jk * NX, j = jk % NY, k = jk / NY;
  const int64_t oi[3] = {i > 0 ? -1 : 0, 0, i < g.nx ? 1 : 0};
  const int64_t oj[3] = {j > 0 ? -NX : 0, 0, j < g.ny ? NX : 0};
  const int64_t ok[3] = {k > 0 ? -NXY : 0, 0, k < g.nz ? NXY : 0};
  const bool in_i[3] = {i > 0, true, i < g.nx};
  const bool in_j[3] = {j > 0, true, j < g.ny};
  const bool in_k[3] = {k > 0, true, k < g.nz};
  double s[3] = {0.0, 0.0, 0.0}, xc[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int slot = 0; slot < 27; ++slot) {
    const int64_t nb = node + oi[slot % 3] + oj[(slot / 3) % 3] + ok[slot / 9];
    const double x0 = x[3 * nb], x1 = x[3 * nb + 1], x2 = x[3 * nb + 2];
    if (slot == 13) {
      xc[0] = x0;
      xc[1] = x1;
      xc[2] = x2;
    }
    double a[9];
    if (slot >= 13) {
      const double* p = Ts + (node >> 5) * (kSymQ * 32) + (slot - 13) * (9 * 32) + (node & 31);
#pragma unroll
      for (int e = 0; e < 9; ++e) a[e] = __ldcs(p + e * 32);
    } else {
      // transpose of the neighbour's mirror block (zero outside the grid,
      // where nb is clamped onto the node itself)
      const bool in = in_i[slot % 3] && in_j[(slot / 3) % 3] && in_k[slot / 9];
      const double* p = Ts + (nb >> 5) * (kSymQ * 32) + (13 - slot) * (9 * 32) + (nb & 31);
#pragma unroll
      for (int ra = 0; ra < 3; ++ra)
#pragma unroll
        for (int cb = 0; cb < 3; ++cb) a[ra * 3 + cb] = in ? __ldg(p + (cb * 3 + ra) * 32) : 0.0;
    }
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      s[r] = __dadd_rn(s[r], __dmul_rn(a[3 * r + 0], x0));
      s[r] = __dadd_rn(s[r], __dmul_rn(a[3 * r + 1], x1));
      s[r] = __dadd_rn(s[r], __dmul_rn(a[3 * r + 2], x2));
    }
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int64_t q = 3 * node + r;
    if (mode == 0) {
      xout[q] = s[r];
    } else if (mode == 2) {
      xout[q] = __dsub_rn(b[q], s[r]);
    } else {
      const double rv = __dsub_rn(b[q], s[r]);
      double dv = __dmul_rn(A, __dmul_rn(dinv[q], rv));
      if (!first) dv = __dadd_rn(dv, __dmul_rn(AC, d[q]));
      d[q] = dv;
      xout[q] = __dadd_rn(xc[r], dv);
    }
  }
}
void stencil_sym64(const Grid& g, const double* Ts, int mode, const double* x, double* out,
                   const double* b, const double* dinv, double* d, double A, double AC, bool first,
                   cudaStream_t s) {
  const int64_t nn = g.d.nnodes();
  stencil_sym_kernel<<<grid_blocks(nn, 128), 128, 0, s>>>(g.d, Ts, x, mode, b, dinv, d, out, A, AC,
                                                          first ? 1 : 0);
  SG_CHECK_LAUNCH();
}

void stencil_cheb64(const Grid& g, const double* At, const double* x, double* xout, const double* b,
                    const double* dinv, double* d, double A, double AC, bool first, cudaStream_t s) {
  const int64_t nn = g.d.nnodes();
  stencil_fused_kernel<<<grid_blocks(nn, 128), 128, 0, s>>>(g.d, At, x, 1, b, dinv, d, xout, A, AC,
                                                            first ? 1 : 0);
  SG_CHECK_LAUNCH();
}
void stencil_res64(const Grid& g, const double* At, const double* x, const double* r, double* out,
                   cudaStream_t s) {
  const int64_t nn = g.d.nnodes();
  stencil_fused_kernel<<<grid_blocks(nn, 128), 128, 0, s>>>(g.d, At, x, 2, r, nullptr, nullptr, out,
                                                            0.0, 0.0, 1);
  SG_CHECK_LAUNCH();
}

template <class T>
void stencil_apply(const Grid& g, const T* At, const T* x, T* y, cudaStream_t s) {
  const int64_t nn = g.d.nnodes();
  stencil_apply_kernel<T><<<grid_blocks(nn, 128), 128, 0, s>>>(g.d, At, x, y);
  SG_CHECK_LAUNCH();
}

// At[(tile*243 + q)*32 + lane] = A[q*nn + tile*32 + lane] (zero padded)
template <class T>
__global__ void stencil_tile_kernel(int64_t nn, int64_t ntiles, const T* __restrict__ A,
                                    T* __restrict__ At) {
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= ntiles * 243 * 32) return;
  const int64_t lane = idx & 31, q = (idx >> 5) % 243, tile = (idx >> 5) / 243;
  const int64_t node = tile * 32 + lane;
  At[idx] = node < nn ? A[q * nn + node] : T(0);
}
template <class T>
void stencil_tile(const Grid& g, const T* A, DBuf<T>& At, cudaStream_t s) {
  const int64_t nn = g.d.nnodes(), nt = (nn + 31) / 32;
  At.alloc(size_t(nt * 243 * 32));
  stencil_tile_kernel<T><<<grid_blocks(nt * 243 * 32, 256), 256, 0, s>>>(nn, nt, A, At.p);
  SG_CHECK_LAUNCH();
}
template void stencil_tile<double>(const Grid&, const double*, DBuf<double>&, cudaStream_t);
template void stencil_tile<float>(const Grid&, const float*, DBuf<float>&, cudaStream_t);
template void stencil_apply<double>(const Grid&, const double*, const double*, double*, cudaStream_t);
template void stencil_apply<float>(const Grid&, const float*, const float*, float*, cudaStream_t);

__global__ void stencil_diag_kernel(int64_t nn, const double* __restrict__ A, double* __restrict__ d) {
  const int64_t node = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (node >= nn) return;
#pragma unroll
  for (int r = 0; r < 3; ++r) d[3 * node + r] = A[int64_t(13 * 9 + r * 3 + r) * nn + node];
}
void stencil_diag(const Grid& g, const double* A, double* d, cudaStream_t s) {
  const int64_t nn = g.d.nnodes();
  stencil_diag_kernel<<<grid_blocks(nn, 256), 256, 0, s>>>(nn, A, d);
  SG_CHECK_LAUNCH();
}

__global__ void round_f32_kernel(int64_t n, const double* __restrict__ a, float* __restrict__ b,
                                 bool bf16) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const float v = __double2float_rn(a[q]);
  b[q] = bf16 ? bf16_round(v) : v;
}
void stencil_round_f32(const Grid& g, const double* A64, float* A32, bool bf16, cudaStream_t s) {
  const int64_t n = 243 * g.d.nnodes();
  round_f32_kernel<<<grid_blocks(n, 256), 256, 0, s>>>(n, A64, A32, bf16);
  SG_CHECK_LAUNCH();
}

// Fine operator as a stencil: A[node][nb] = sum over elements e containing
// both (ascending e) of E_e * Ke[3a+ra][3b+cb], FMA-free -- the same sum as
// FineOperator.assemble_dense (fine_operator.py:88-101).
__global__ void fine_to_stencil_kernel(GridDesc g, const uint8_t* __restrict__ nmask,
                                       const double* __restrict__ E, KeParam<double> ke,
                                       double* __restrict__ A) {
  const int64_t nn = g.nnodes();
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= nn * 27) return;
  const int64_t node = q % nn;
  const int slot = int(q / nn);
  const int di = slot % 3 - 1, dj = (slot / 3) % 3 - 1, dk = slot / 9 - 1;
  const int NX = g.nx + 1, NY = g.ny + 1;
  const int i = int(node % NX), j = int((node / NX) % NY), k = int(node / (int64_t(NX) * NY));
  double acc[9];
#pragma unroll
  for (int t = 0; t < 9; ++t) acc[t] = 0.0;
  const int ni = i + di, nj = j + dj, nk = k + dk;
  const bool nb_ok = ni >= 0 && ni <= g.nx && nj >= 0 && nj <= g.ny && nk >= 0 && nk <= g.nz;
  if (nb_ok) {
    const int64_t nb = ni + int64_t(NX) * (nj + int64_t(NY) * nk);
    for (int ek = k - 1; ek <= k; ++ek) {
      if (ek < 0 || ek >= g.nz || nk < ek || nk > ek + 1) continue;
      for (int ej = j - 1; ej <= j; ++ej) {
        if (ej < 0 || ej >= g.ny || nj < ej || nj > ej + 1) continue;
        for (int ei = i - 1; ei <= i; ++ei) {
          if (ei < 0 || ei >= g.nx || ni < ei || ni > ei + 1) continue;
          const int64_t e = ei + int64_t(g.nx) * (ej + int64_t(g.ny) * ek);
          const int a = (i - ei) + 2 * (j - ej) + 4 * (k - ek);
          const int b = (ni - ei) + 2 * (nj - ej) + 4 * (nk - ek);
          const double ev = E[e];
#pragma unroll
          for (int ra = 0; ra < 3; ++ra)
#pragma unroll
            for (int cb = 0; cb < 3; ++cb)
              acc[ra * 3 + cb] = __dadd_rn(acc[ra * 3 + cb], __dmul_rn(ev, ke.k[(3 * a + ra) * 24 + 3 * b + cb]));
        }
      }
    }
#pragma unroll
    for (int ra = 0; ra < 3; ++ra)
#pragma unroll
      for (int cb = 0; cb < 3; ++cb)
        if (node_fixed_axis(g, nmask, node, i, ra) || node_fixed_axis(g, nmask, nb, ni, cb))
          acc[ra * 3 + cb] = 0.0;
  }
#pragma unroll
  for (int t = 0; t < 9; ++t) A[(int64_t(slot) * 9 + t) * nn + node] = acc[t];
}
void fine_to_stencil(const FineOp& op, double* A, cudaStream_t s) {
  const int64_t n = 27 * op.grid.d.nnodes();
  fine_to_stencil_kernel<<<grid_blocks(n, 128), 128, 0, s>>>(op.grid.d, op.grid.nmask.p, op.E64.p,
                                                             op.ke64, A);
  SG_CHECK_LAUNCH();
}

// ---------------------------------------------------------------- export
__device__ __forceinline__ bool slot_neighbor(const GridDesc& g, int64_t node, int slot, int64_t* nb) {
  const int NX = g.nx + 1, NY = g.ny + 1;
  const int i = int(node % NX), j = int((node / NX) % NY), k = int(node / (int64_t(NX) * NY));
  const int di = slot % 3 - 1, dj = (slot / 3) % 3 - 1, dk = slot / 9 - 1;
  if (i + di < 0 || i + di > g.nx || j + dj < 0 || j + dj > g.ny || k + dk < 0 || k + dk > g.nz)
    return false;
  *nb = node + di + int64_t(NX) * (dj + int64_t(NY) * dk);
  return true;
}

__global__ void row_count_kernel(GridDesc g, int64_t nfree, const int32_t* __restrict__ f2d,
                                 const int32_t* __restrict__ d2f, const double* __restrict__ A,
                                 int64_t* __restrict__ counts) {
  const int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (f >= nfree) return;
  const int64_t nn = g.nnodes();
  const int64_t node = f2d[f] / 3;
  const int ra = f2d[f] % 3;
  int64_t c = 0;
  for (int slot = 0; slot < 27; ++slot) {
    int64_t nb;
    if (!slot_neighbor(g, node, slot, &nb)) continue;
    for (int cb = 0; cb < 3; ++cb)
      if (d2f[3 * nb + cb] >= 0 && A[(int64_t(slot) * 9 + ra * 3 + cb) * nn + node] != 0.0) ++c;
  }
  counts[f] = c;
}

__global__ void row_fill_kernel(GridDesc g, int64_t nfree, const int32_t* __restrict__ f2d,
                                const int32_t* __restrict__ d2f, const double* __restrict__ A,
                                const int64_t* __restrict__ indptr, int64_t* __restrict__ indices,
                                double* __restrict__ data) {
  const int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (f >= nfree) return;
  const int64_t nn = g.nnodes();
  const int64_t node = f2d[f] / 3;
  const int ra = f2d[f] % 3;
  int64_t o = indptr[f];
  for (int slot = 0; slot < 27; ++slot) {
    int64_t nb;
    if (!slot_neighbor(g, node, slot, &nb)) continue;
    for (int cb = 0; cb < 3; ++cb) {
      const double v = A[(int64_t(slot) * 9 + ra * 3 + cb) * nn + node];
      if (d2f[3 * nb + cb] >= 0 && v != 0.0) {
        indices[o] = d2f[3 * nb + cb];
        data[o] = v;
        ++o;
      }
    }
  }
}

static void row_counts(const Grid& g, const double* A, std::vector<int64_t>& indptr, cudaStream_t s) {
  DBuf<int64_t> cnt{size_t(std::max<int64_t>(g.n_free, 1))};
  row_count_kernel<<<grid_blocks(g.n_free, 128), 128, 0, s>>>(g.d, g.n_free, g.free2dof.p,
                                                              g.dof2free.p, A, cnt.p);
  SG_CHECK_LAUNCH();
  std::vector<int64_t> h(static_cast<size_t>(size_t(g.n_free)));
  cnt.download(h.data(), h.size(), s);
  SG_CUDA(cudaStreamSynchronize(s));
  indptr.assign(size_t(g.n_free + 1), 0);
  for (int64_t f = 0; f < g.n_free; ++f) indptr[f + 1] = indptr[f] + h[f];
}

int64_t stencil_count_nnz(const Grid& g, const double* A, cudaStream_t s) {
  if (!g.n_free) return 0;
  std::vector<int64_t> indptr;
  row_counts(g, A, indptr, s);
  return indptr.back();
}

void stencil_export_csr(const Grid& g, const double* A, int64_t* indptr_h, int64_t* indices_h,
                        double* data_h, cudaStream_t s) {
  std::vector<int64_t> indptr;
  if (!g.n_free) {
    indptr_h[0] = 0;
    return;
  }
  row_counts(g, A, indptr, s);
  const int64_t nnz = indptr.back();
  DBuf<int64_t> dptr(indptr.size()), dind(size_t(std::max<int64_t>(nnz, 1)));
  DBuf<double> ddat{size_t(std::max<int64_t>(nnz, 1))};
  dptr.upload(indptr.data(), indptr.size(), s);
  row_fill_kernel<<<grid_blocks(g.n_free, 128), 128, 0, s>>>(g.d, g.n_free, g.free2dof.p,
                                                             g.dof2free.p, A, dptr.p, dind.p, ddat.p);
  SG_CHECK_LAUNCH();
  dind.download(indices_h, size_t(nnz), s);
  ddat.download(data_h, size_t(nnz), s);
  SG_CUDA(cudaStreamSynchronize(s));
  std::copy(indptr.begin(), indptr.end(), indptr_h);
}

__global__ void dense_kernel(GridDesc g, int64_t nfree, const int32_t* __restrict__ f2d,
                             const int32_t* __restrict__ d2f, const double* __restrict__ A,
                             double eps, double* __restrict__ D) {
  const int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (f >= nfree) return;
  const int64_t nn = g.nnodes();
  const int64_t node = f2d[f] / 3;
  const int ra = f2d[f] % 3;
  double* row = D + f * nfree;
  for (int slot = 0; slot < 27; ++slot) {
    int64_t nb;
    if (!slot_neighbor(g, node, slot, &nb)) continue;
    for (int cb = 0; cb < 3; ++cb) {
      const int32_t c = d2f[3 * nb + cb];
      if (c >= 0) row[c] = A[(int64_t(slot) * 9 + ra * 3 + cb) * nn + node];
    }
  }
  row[f] = row[f] + eps;
}
void stencil_to_dense(const Grid& g, const double* A, double* D, double eps, cudaStream_t s) {
  SG_CUDA(cudaMemsetAsync(D, 0, sizeof(double) * g.n_free * g.n_free, s));
  dense_kernel<<<grid_blocks(g.n_free, 128), 128, 0, s>>>(g.d, g.n_free, g.free2dof.p,
                                                          g.dof2free.p, A, eps, D);
  SG_CHECK_LAUNCH();
}

}  // namespace sg
