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

int kKwRowHost(int q) { return kKwRowH[q]; }
int kKwColHost(int q) { return kKwColH[q]; }

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
__global__ void __launch_bounds__(kWThreads, 2)
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
  // predicates; running pointers advance one node plane per layer.
  const int ci0 = min(max(ei, 0), g.nx), ci1 = min(max(ei + 1, 0), g.nx);
  const int cj0 = min(max(ej, 0), g.ny), cj1 = min(max(ej + 1, 0), g.ny);
  const int off1 = 3 * (ci1 - ci0), off2 = 3 * NX * (cj1 - cj0);
  const int64_t plane = 3 * int64_t(NX) * NY;
  const T* ucol = u + 3 * (int64_t(ci0) + int64_t(NX) * cj0);
  const T* ulast = ucol + int64_t(g.nz) * plane;
  const int64_t estride = int64_t(g.nx) * g.ny;
  const T* ecol = E + (col_in ? ei + int64_t(g.nx) * ej : 0);
  // per-thread constants of the owned node column
  const bool xface_fixed = g.xface && ni == 0;
  T* yp = y + 3 * (int64_t(min(ni, g.nx)) + int64_t(NX) * min(nj, g.ny)) + int64_t(k0) * plane;
  const uint8_t* mp = nmask ? nmask + (int64_t(min(ni, g.nx)) + int64_t(NX) * min(nj, g.ny)) +
                                  int64_t(k0) * NX * NY : nullptr;

  auto load_plane = [&](const T* p, T* dst) {
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
  const T* pnext = ucol + int64_t(max(k0 - 1, 0)) * plane;

  T carry[3] = {T(0), T(0), T(0)};
  int buf = 0;

  // one element layer: lo = plane ek, hi = plane ek+1 (corners 0..3 each)
  auto layer = [&](int ek, const T* lo, const T* hi, T s) {
    T v[24];
    // forward Walsh on the 2x2x2 corners, built from lo/hi without copies
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const T a0 = lo[c], a1 = lo[3 + c], a2 = lo[6 + c], a3 = lo[9 + c];
      const T a4 = hi[c], a5 = hi[3 + c], a6 = hi[6 + c], a7 = hi[9 + c];
      const T b0 = a0 + a1, b1 = a0 - a1, b2 = a2 + a3, b3 = a2 - a3;
      const T b4 = a4 + a5, b5 = a4 - a5, b6 = a6 + a7, b7 = a6 - a7;
      const T c0 = b0 + b2, c2 = b0 - b2, c1 = b1 + b3, c3 = b1 - b3;
      const T c4 = b4 + b6, c6 = b4 - b6, c5 = b5 + b7, c7 = b5 - b7;
      v[c] = T(0);  // constant mode: rigid translation, no energy
      v[3 + c] = c1 + c5;
      v[6 + c] = c2 + c6;
      v[9 + c] = c3 + c7;
      v[12 + c] = c0 - c4;
      v[15 + c] = c1 - c5;
      v[18 + c] = c2 - c6;
      v[21 + c] = c3 - c7;
    }
    T w[24];
#pragma unroll
    for (int r = 0; r < 24; ++r) w[r] = T(0);
#pragma unroll
    for (int q = 0; q < 45; ++q) w[kKwRow[q]] += P.v[q] * v[kKwCol[q]];
#pragma unroll
    for (int r = 3; r < 24; ++r) w[r] *= s;
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
    for (int t = 0; t < 6; ++t) ex[buf][ty][tx][t] = A[t];
    __syncthreads();
    T B[6];
    const bool up = ty < kWY - 1;
#pragma unroll
    for (int t = 0; t < 6; ++t) B[t] = up ? A[6 + t] + ex[buf][ty + 1][tx][t] : A[6 + t];
    buf ^= 1;
    // z-combine: node plane ek = carry (top of layer ek-1) + bottom of layer ek
    if (ek >= k0) {
      if (own) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const bool fixed = g.xface ? xface_fixed : ((mp[0] >> c) & 1);
          yp[c] = fixed ? T(0) : carry[c] + B[c];
        }
      }
      yp += plane;
      if (!g.xface) mp += int64_t(NX) * NY;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) carry[c] = B[3 + c];
  };

  // three rotating plane buffers: the plane two layers ahead is in flight
  // while the current element is computed
  T QA[12], QB[12], QC[12];
  load_plane(pnext, QA);  // plane k0-1 (clamped)
  pnext = ucol + int64_t(min(max(k0, 0), g.nz)) * plane;
  load_plane(pnext, QB);  // plane k0
  T sA = load_E(k0 - 1);
  for (int ek = k0 - 1; ek < k1; ek += 3) {
    pnext = pnext < ulast ? pnext + plane : ulast;
    load_plane(pnext, QC);
    T sB = load_E(ek + 1);
    layer(ek, QA, QB, sA);
    if (ek + 1 >= k1) break;
    pnext = pnext < ulast ? pnext + plane : ulast;
    load_plane(pnext, QA);
    T sC = load_E(ek + 2);
    layer(ek + 1, QB, QC, sB);
    if (ek + 2 >= k1) break;
    pnext = pnext < ulast ? pnext + plane : ulast;
    load_plane(pnext, QB);
    sA = load_E(ek + 3);
    layer(ek + 2, QC, QA, sC);
  }
}

template <class T>
static void launch_walsh(const FineOp& op, const T* u, T* y, const T* E, const KwParam<T>& P,
                         cudaStream_t s) {
  const GridDesc& g = op.grid.d;
  const int tx = (g.nx + 1 + kWX - 2) / (kWX - 1);
  const int ty = (g.ny + 1 + kWY - 2) / (kWY - 1);
  const int planes = g.nz + 1;
  // z-chunking: minimise the busiest SM's layer count, (CTAs per SM) x
  // (layers per chunk incl. the halo layer), at two resident CTAs per SM
  int best = 1, best_cost = 1 << 30;
  for (int nc = 1; nc <= std::max(1, planes / 4); ++nc) {
    const int kc = (planes + nc - 1) / nc;
    const int n = (planes + kc - 1) / kc;
    const int ctas = tx * ty * n;
    const int waves = (ctas + 2 * num_sms() - 1) / (2 * num_sms());
    const int per_sm = (ctas + num_sms() - 1) / num_sms();
    const int cost = std::max(per_sm, 2 * waves) * (kc + 1);
    if (cost < best_cost) { best_cost = cost; best = n; }
  }
  const int kchunk = (planes + best - 1) / best;
  const int nchunk = (planes + kchunk - 1) / kchunk;
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
