// Level-0 matrix-free apply, flop-reduced and z-streaming (FP32 / FP64).
//
// In the tensor Walsh basis (per displacement component, corner c = x+2y+4z,
// W[m][c] = (-1)^popcount(m&c)) the unit Q1 stiffness has 45 nonzeros out of
// 576, so y_e = (E_e/64) * W (Kw (W u_e)) costs ~210 flops per element
// instead of 1152 -- bringing the FP32 apply below the B200's
// FP32 ridge so it can run at the HBM roofline.
//
// Work decomposition: a CTA owns a 15 x 15 column of nodes (16 x 16 element
// columns incl. one halo element per direction) and a chunk of z-planes; it
// streams element layers upward.  Per layer a thread evaluates one element;
// the 8 corner results are combined deterministically (no atomics):
// x-neighbour by a warp shuffle, y-neighbour through shared memory, and the
// two z-layers sharing a node plane in registers.  Each node therefore sums
// its 8 elements in a fixed order, run-to-run bit-reproducible.
#include "sg_kernels.cuh"

namespace sg {

// 45-entry sparsity pattern of W Ke W (index = 3*mode + component); the
// values are computed on the host from the same Ke (walsh_params()).
__device__ constexpr int kKwRow[45] = {3, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 7, 8, 8, 9,
                                       9, 10, 10, 11, 11, 11, 12, 12, 13, 13, 14, 14, 14, 15, 15,
                                       16, 16, 16, 17, 17, 18, 18, 18, 19, 19, 20, 20, 21, 22, 23};
__device__ constexpr int kKwCol[45] = {3, 7, 14, 4, 6, 5, 12, 4, 6, 3, 7, 14, 8, 13, 9,
                                       20, 10, 17, 11, 16, 18, 5, 12, 8, 13, 3, 7, 14, 15, 19,
                                       11, 16, 18, 10, 17, 11, 16, 18, 15, 19, 9, 20, 21, 22, 23};
const int kKwRowH[45] = {3, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 7, 8, 8, 9,
                         9, 10, 10, 11, 11, 11, 12, 12, 13, 13, 14, 14, 14, 15, 15,
                         16, 16, 16, 17, 17, 18, 18, 18, 19, 19, 20, 20, 21, 22, 23};
const int kKwColH[45] = {3, 7, 14, 4, 6, 5, 12, 4, 6, 3, 7, 14, 8, 13, 9,
                         20, 10, 17, 11, 16, 18, 5, 12, 8, 13, 3, 7, 14, 15, 19,
                         11, 16, 18, 10, 17, 11, 16, 18, 15, 19, 9, 20, 21, 22, 23};

bool walsh_params(const double* ke, KwParam<double>& p64, KwParam<float>& p32) {
  double Kw[24][24];
  double maxabs = 0.0;
  for (int r = 0; r < 24; ++r)
    for (int c = 0; c < 24; ++c) {
      if (r % 3 != 0 && false) {}
      double s = 0.0;
      const int mr = r / 3, ar = r % 3, mc = c / 3, ac = c % 3;
      for (int a = 0; a < 8; ++a)
        for (int b = 0; b < 8; ++b) {
          const double wa = (__builtin_popcount(mr & a) & 1) ? -1.0 : 1.0;
          const double wb = (__builtin_popcount(mc & b) & 1) ? -1.0 : 1.0;
          s += wa * ke[(3 * a + ar) * 24 + 3 * b + ac] * wb;
        }
      Kw[r][c] = s;
      maxabs = std::max(maxabs, std::fabs(s));
    }
  bool in_pat[24][24] = {};
  for (int q = 0; q < 45; ++q) {
    in_pat[kKwRowH[q]][kKwColH[q]] = true;
    p64.v[q] = Kw[kKwRowH[q]][kKwColH[q]] / 64.0;
    p32.v[q] = float(p64.v[q]);
  }
  for (int r = 0; r < 24; ++r)
    for (int c = 0; c < 24; ++c)
      if (!in_pat[r][c] && std::fabs(Kw[r][c]) > 1e-12 * maxabs) return false;
  return true;
}

template <class T>
__device__ __forceinline__ void fwht8(T* v) {  // in-place unnormalised Walsh, stride 3
#pragma unroll
  for (int b = 1; b < 8; b <<= 1)
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (!(c & b)) {
        const T a = v[3 * c], d = v[3 * (c | b)];
        v[3 * c] = a + d;
        v[3 * (c | b)] = a - d;
      }
}

template <class T>
__device__ __forceinline__ T shfl_down16(T v) {
  return __shfl_down_sync(0xffffffffu, v, 1, 16);
}

constexpr int kWX = 16;   // element columns per tile along x (15 owned nodes)
constexpr int kWY = 16;   // element columns per tile along y (15 owned nodes)
constexpr int kWThreads = kWX * kWY;

template <class T>
__global__ void __launch_bounds__(kWThreads, sizeof(T) == 4 ? 3 : 1)
fine_apply_walsh_kernel(GridDesc g, const uint8_t* __restrict__ nmask, const T* __restrict__ u,
                        T* __restrict__ y, const T* __restrict__ E, KwParam<T> P, int kchunk) {
  __shared__ T ex[2][kWY][kWX][6];
  const int tx = threadIdx.x & (kWX - 1);
  const int ty = threadIdx.x / kWX;
  const int ei = int(blockIdx.x) * (kWX - 1) - 1 + tx;
  const int ej = int(blockIdx.y) * (kWY - 1) - 1 + ty;
  const int k0 = int(blockIdx.z) * kchunk;
  const int k1 = min(k0 + kchunk, g.nz + 1);  // output node planes [k0, k1)
  const int NX = g.nx + 1, NY = g.ny + 1;
  const int ni = ei + 1, nj = ej + 1;         // owned node column (upper corner)
  const bool own = tx < kWX - 1 && ty < kWY - 1 && ni <= g.nx && nj <= g.ny;
  const bool col_in = ei >= 0 && ei < g.nx && ej >= 0 && ej < g.ny;
  // Corner loads use clamped (always valid) addresses: a corner is only ever
  // out of the domain for an element that is itself outside, and those get
  // modulus 0, so their (finite) inputs never reach a result.  No per-load
  // predicates, one pointer bump per plane.
  const int ci0 = min(max(ei, 0), g.nx), ci1 = min(max(ei + 1, 0), g.nx);
  const int cj0 = min(max(ej, 0), g.ny), cj1 = min(max(ej + 1, 0), g.ny);
  const int off1 = 3 * (ci1 - ci0), off2 = 3 * NX * (cj1 - cj0);
  const int64_t plane = 3 * int64_t(NX) * NY;
  const T* ucol = u + 3 * (int64_t(ci0) + int64_t(NX) * cj0);
  const int64_t estride = int64_t(g.nx) * g.ny;
  const T* ecol = E + (col_in ? ei + int64_t(g.nx) * ej : 0);
  auto load_plane = [&](int kp, T* dst) {
    const T* p = ucol + int64_t(min(max(kp, 0), g.nz)) * plane;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      dst[c] = __ldg(p + c);
      dst[3 + c] = __ldg(p + off1 + c);
      dst[6 + c] = __ldg(p + off2 + c);
      dst[9 + c] = __ldg(p + off2 + off1 + c);
    }
  };
  auto load_E = [&](int ek) {
    const bool el_ok = col_in && ek >= 0 && ek < g.nz;
    const T e = __ldg(ecol + int64_t(min(max(ek, 0), g.nz - 1)) * estride);
    return el_ok ? e : T(0);
  };

  T lo[12];  // u at the lower node plane of the current layer (corners 0..3)
  load_plane(k0 - 1, lo);
  T carry[3] = {T(0), T(0), T(0)};
  int buf = 0;
  // software pipeline: the upper plane of layer ek and its modulus are loaded
  // one iteration ahead, so the global-load latency overlaps the element math
  T hi[12];
  T s_next;
  load_plane(k0, hi);
  s_next = load_E(k0 - 1);
  for (int ek = k0 - 1; ek < k1; ++ek) {
    T v[24];
#pragma unroll
    for (int q = 0; q < 12; ++q) {
      v[(q / 3) * 3 + q % 3] = lo[q];
      v[12 + q] = hi[q];
      lo[q] = hi[q];
    }
    const T s = s_next;
    if (ek + 1 < k1) {
      load_plane(ek + 2, hi);
      s_next = load_E(ek + 1);
    }
    // forward Walsh per component
#pragma unroll
    for (int c = 0; c < 3; ++c) fwht8(v + c);
    // sparse core: w = s * Kw v  (constant modes 0..2 stay zero)
    T w[24];
#pragma unroll
    for (int r = 0; r < 24; ++r) w[r] = T(0);
#pragma unroll
    for (int q = 0; q < 45; ++q) w[kKwRow[q]] += P.v[q] * v[kKwCol[q]];
#pragma unroll
    for (int r = 3; r < 24; ++r) w[r] *= s;
    // inverse Walsh per component -> 8 corner results
#pragma unroll
    for (int c = 0; c < 3; ++c) fwht8(w + c);
    // x-combine: node (ei+1, ej+jy, ek+kz) <- own corner (1,jy,kz) + right corner (0,jy,kz)
    T A[12];
#pragma unroll
    for (int jy = 0; jy < 2; ++jy)
#pragma unroll
      for (int kz = 0; kz < 2; ++kz)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int cr = 1 + 2 * jy + 4 * kz, cl = 2 * jy + 4 * kz;
          A[(jy * 2 + kz) * 3 + c] = w[3 * cr + c] + shfl_down16(w[3 * cl + c]);
        }
    // y-combine through shared memory: node row ej+1 <- own jy=1 + upper thread's jy=0
#pragma unroll
    for (int t = 0; t < 6; ++t) ex[buf][ty][tx][t] = A[t];  // jy = 0 entries (kz, c)
    __syncthreads();
    T B[6];
    if (ty < kWY - 1) {
#pragma unroll
      for (int t = 0; t < 6; ++t) B[t] = A[6 + t] + ex[buf][ty + 1][tx][t];
    } else {
#pragma unroll
      for (int t = 0; t < 6; ++t) B[t] = A[6 + t];
    }
    buf ^= 1;
    // z-combine: node plane ek = carry (top of layer ek-1) + bottom of layer ek
    if (ek >= k0 && own) {
      const int64_t node = ni + int64_t(NX) * (nj + int64_t(NY) * ek);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const T val = carry[c] + B[c];
        y[3 * node + c] = node_fixed_axis(g, nmask, node, ni, c) ? T(0) : val;
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) carry[c] = B[3 + c];
  }
}

template <class T>
static void launch_walsh(const FineOp& op, const T* u, T* y, const T* E, const KwParam<T>& P,
                         cudaStream_t s) {
  const GridDesc& g = op.grid.d;
  const int tx = (g.nx + 1 + kWX - 2) / (kWX - 1);
  const int ty = (g.ny + 1 + kWY - 2) / (kWY - 1);
  const int planes = g.nz + 1;
  // about two CTAs per SM in total, chunks of at least 8 planes
  int nchunk = (2 * kNumSMs + tx * ty - 1) / (tx * ty);
  nchunk = std::max(1, std::min(nchunk, (planes + 7) / 8));
  const int kchunk = (planes + nchunk - 1) / nchunk;
  nchunk = (planes + kchunk - 1) / kchunk;
  dim3 grid(tx, ty, nchunk);
  fine_apply_walsh_kernel<T><<<grid, kWThreads, 0, s>>>(g, op.grid.nmask.p, u, y, E, P, kchunk);
  SG_CHECK_LAUNCH();
}

void fine_apply_walsh_f32(const FineOp& op, const float* u, float* y, cudaStream_t s) {
  launch_walsh<float>(op, u, y, op.E32.p, op.kw32, s);
}
void fine_apply_walsh_f64(const FineOp& op, const double* u, double* y, cudaStream_t s) {
  launch_walsh<double>(op, u, y, op.E64.p, op.kw64, s);
}

}  // namespace sg
