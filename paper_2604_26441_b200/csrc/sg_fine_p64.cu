// Level-0 matrix-free FP64 apply on node-layout vectors (fine_operator.py:61-67,
// the outer PCG's K p every iteration, krylov.py:136).
//
// Same algebra as the packed FP32 kernel (sg_fine_pk.cu): tensor Walsh basis,
// the 45-entry Kw in its block form (33 ops + 8 coefficient scalings per
// element instead of 45 + 21), the x/y stage of a node plane computed once and
// shared by the element layers below and above it, and the two layers sharing
// a node plane added in the Walsh-xy domain before the xy inverse.  FP64 has
// no packed form, so a thread owns ONE element and streams it up a z-chunk.
//  * tile: R element rows x W element columns flattened (t = row*W + col),
//    W - 1 node columns and R - 1 node rows owned (one recomputed halo
//    element per direction), a z-chunk of node planes (+ one recomputed
//    layer); W chosen so the x tiles split NX evenly (pk64_plan);
//  * node planes are staged in shared memory by cooperative coalesced loads
//    of whole node-layout rows ((W+1) nodes x 3 components contiguous), one
//    plane ahead in registers: the 24-byte node stride never reaches the
//    LSU as strided scalar loads;
//  * neighbour partial sums through shared memory (one barrier per layer) in a
//    fixed order: node (i, j) = (own + right) + (up + up-right), the same for
//    every tiling -> bit-identical on slab windows and run to run.
#include <cmath>
#include <cstdlib>
#include "sg_kernels.cuh"

namespace sg {

constexpr int kP64MaxThreads = 512;

struct PkCoefD {
  double amb, b, c, d, e, fmg, g, h;
};

// Kw/64 block parameters in FP64 (see pk_params in sg_fine_pk.cu for the
// block structure; false = Ke lacks it and the scalar Walsh kernel runs).
static bool pk64_params(const FineOp& op, PkCoefD& C) {
  double Kw[24][24] = {};
  for (int q = 0; q < 45; ++q) Kw[kKwRowHost(q)][kKwColHost(q)] = op.kw64.v[q];
  const double a = Kw[3][3], b = Kw[3][7], c = Kw[4][4], d = Kw[9][9], e = Kw[9][20],
               f = Kw[11][11], gg = Kw[11][16], h = Kw[21][21];
  double want[24][24] = {};
  auto blk3 = [&](int i, int j, int k, double p, double q) {
    const int id[3] = {i, j, k};
    for (int r = 0; r < 3; ++r)
      for (int s = 0; s < 3; ++s) want[id[r]][id[s]] = r == s ? p : q;
  };
  auto blk2 = [&](int i, int j, double p, double q) {
    want[i][i] = want[j][j] = p;
    want[i][j] = want[j][i] = q;
  };
  blk3(3, 7, 14, a, b);
  blk3(11, 16, 18, f, gg);
  blk2(4, 6, c, c);
  blk2(5, 12, c, c);
  blk2(8, 13, c, c);
  blk2(9, 20, d, e);
  blk2(10, 17, d, e);
  blk2(15, 19, d, e);
  want[21][21] = want[22][22] = want[23][23] = h;
  double mx = 0.0;
  for (int r = 0; r < 24; ++r)
    for (int s = 0; s < 24; ++s) mx = std::max(mx, std::fabs(Kw[r][s]));
  for (int r = 0; r < 24; ++r)
    for (int s = 0; s < 24; ++s)
      if (std::fabs(Kw[r][s] - want[r][s]) > 1e-12 * mx) return false;
  C.amb = a - b;
  C.b = b;
  C.c = c;
  C.d = d;
  C.e = e;
  C.fmg = f - gg;
  C.g = gg;
  C.h = h;
  return true;
}

// NT: compile-time block size (0: runtime); 256-thread blocks run two CTAs
// per SM (NT = 256 -> __launch_bounds__(256, 2))
constexpr int p64_bs(int nt) { return nt > 0 ? nt : kP64MaxThreads; }
template <int LD, int NT>
__global__ void __launch_bounds__(p64_bs(NT), kP64MaxThreads / p64_bs(NT))
fine_p64_kernel(GridDesc g, const uint8_t* __restrict__ nmask, const double* __restrict__ u,
                double* __restrict__ yout, const double* __restrict__ E, PkCoefD C, int W, int R,
                int kchunk) {
  // shared memory: slab[2][R+1][3(W+1)] node planes (rows y0-1 .. y0+R-1,
  // columns x0-1 .. x0+W-1), pub[2][9][nt] partials, ost[2][R-1][3(W-1)]
  // owned outputs (written back by coalesced row stores one layer later)
  extern __shared__ double p64sm[];
  const int SW = 3 * (W + 1);
  const int SL = (R + 1) * SW;
  const int OW = 3 * (W - 1);
  const int OL = (R - 1) * OW;
  const int nt = NT > 0 ? NT : int(blockDim.x);  // NT: compile-time block size (constant offsets)
  double* slab = p64sm;
  double* pub = slab + 2 * SL;
  double* ost = pub + 18 * nt;
  const int t = threadIdx.x;
  const int row = t / W, col = t - row * W;
  const bool live = row < R;
  const int NX = g.nx + 1, NY = g.ny + 1;
  const int x0 = int(blockIdx.x) * (W - 1);  // first owned node column
  const int y0 = int(blockIdx.y) * (R - 1);  // first owned node row
  const int ex = x0 - 1 + col, ej = y0 - 1 + row;
  const int k0 = int(blockIdx.z) * kchunk;
  const int k1 = min(k0 + kchunk, g.nz + 1);  // output node planes [k0, k1)
  const int64_t plane = int64_t(3) * NX * NY;

  // per-thread slab entries t + i*nt (load offsets within a plane) and owned
  // output entries (store offsets, -1 outside the grid); fixed for the launch
  int gin[LD], gout[LD];
#pragma unroll
  for (int i = 0; i < LD; ++i) {
    const int idx = t + i * nt;
    gin[i] = -1;
    gout[i] = -1;
    if (idx < SL) {
      const int r = idx / SW, q = idx - r * SW, n = q / 3, c = q - 3 * n;
      const int gx = min(max(x0 - 1 + n, 0), g.nx), gy = min(max(y0 - 1 + r, 0), g.ny);
      gin[i] = 3 * (gx + NX * gy) + c;
    }
    if (idx < OL) {
      const int r = idx / OW, q = idx - r * OW, n = q / 3, c = q - 3 * n;
      if (x0 + n <= g.nx && y0 + r <= g.ny) gout[i] = 3 * ((x0 + n) + NX * (y0 + r)) + c;
    }
  }
  double pre[LD];
  auto load_plane = [&](int k) {  // node plane k (clamped) into registers
    const double* p = u + int64_t(min(max(k, 0), g.nz)) * plane;
#pragma unroll
    for (int i = 0; i < LD; ++i) pre[i] = gin[i] >= 0 ? __ldg(p + gin[i]) : 0.0;
  };
  auto store_plane = [&](int buf) {
#pragma unroll
    for (int i = 0; i < LD; ++i)
      if (gin[i] >= 0) slab[buf * SL + t + i * nt] = pre[i];
  };
  auto flush = [&](int ob, int64_t op) {  // owned outputs of plane op -> y
    double* yp = yout + op * plane;
#pragma unroll
    for (int i = 0; i < LD; ++i)
      if (gout[i] >= 0) yp[gout[i]] = ost[ob * OL + t + i * nt];
  };

  const bool rowin = live && ej >= 0 && ej < g.ny && ex >= 0 && ex < g.nx;
  const double* Ep = E + (int64_t(g.nx) * min(max(ej, 0), g.ny - 1) + min(max(ex, 0), g.nx - 1));
  const int64_t estride = int64_t(g.nx) * g.ny;
  auto load_E = [&](int ek) { return __ldg(Ep + int64_t(min(max(ek, 0), g.nz - 1)) * estride); };

  // ownership: node (ex+1, ej+1) = (x0 + col, y0 + row)
  const int oi = ex + 1, oj = ej + 1;
  const bool own = live && col < W - 1 && row < R - 1 && oi <= g.nx && oj <= g.ny;
  const int64_t onode = int64_t(min(oi, g.nx)) + int64_t(NX) * min(oj, g.ny);
  const int lc = min(col, W - 1), lr = min(row, R - 1);  // slab corner (lc, lr) = node (ex, ej)
  const int oidx = min(row, R - 2) * OW + 3 * min(col, W - 2);

  auto plane_q = [&](int buf, double (&Q)[3][4]) {
    const double* s0 = slab + buf * SL + lr * SW + 3 * lc;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double a00 = s0[c], a01 = s0[3 + c], a10 = s0[SW + c], a11 = s0[SW + 3 + c];
      const double S0 = a00 + a01, D0 = a00 - a01, S1 = a10 + a11, D1 = a10 - a11;
      Q[c][0] = S0 + S1;
      Q[c][2] = S0 - S1;
      Q[c][1] = D0 + D1;
      Q[c][3] = D0 - D1;
    }
  };

  double QA[3][4], QB[3][4], carry[3][4];
  // prologue: planes k0-1 (buffer 0) and k0 (buffer 1) staged, k0+1 in flight
  load_plane(k0 - 1);
  store_plane(0);
  load_plane(k0);
  store_plane(1);
  load_plane(k0 + 1);
  __syncthreads();
  plane_q(0, QA);
  __syncthreads();  // buffer 0 is refilled by the first layer's store_plane
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int m = 0; m < 4; ++m) carry[c][m] = 0.0;
  double Ecur = load_E(k0 - 1);
  int pb = 0;  // published-partials / output-stage buffer

  // one element layer ek: node planes ek (Ql, already transformed) and ek+1
  auto layer = [&](int ek, double (&Ql)[3][4], double (&Qh)[3][4]) {
    const int cur = (ek - k0) & 1;  // buffer of node plane ek+1 (plane k in (k - k0 + 1) & 1)
    plane_q(cur, Qh);
    const double En = load_E(ek + 1);
    const bool kin = ek >= 0 && ek < g.nz;
    const double Es = (kin && rowin) ? Ecur : 0.0;
    Ecur = En;
    const double kA = Es * C.amb, kB = Es * C.b, kC = Es * C.c, kD = Es * C.d;
    const double kE = Es * C.e, kF = Es * C.fmg, kG = Es * C.g, kH = Es * C.h;
    double v[24];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
#pragma unroll
      for (int m = 1; m < 4; ++m) v[3 * m + c] = Ql[c][m] + Qh[c][m];
#pragma unroll
      for (int m = 0; m < 4; ++m) v[3 * (m + 4) + c] = Ql[c][m] - Qh[c][m];
    }
    double w[24];
    {
      const double t1 = kB * ((v[3] + v[7]) + v[14]);
      w[3] = fma(kA, v[3], t1);
      w[7] = fma(kA, v[7], t1);
      w[14] = fma(kA, v[14], t1);
      w[4] = w[6] = kC * (v[4] + v[6]);
      w[5] = w[12] = kC * (v[5] + v[12]);
      w[8] = w[13] = kC * (v[8] + v[13]);
      w[9] = fma(kD, v[9], kE * v[20]);
      w[20] = fma(kD, v[20], kE * v[9]);
      w[10] = fma(kD, v[10], kE * v[17]);
      w[17] = fma(kD, v[17], kE * v[10]);
      w[15] = fma(kD, v[15], kE * v[19]);
      w[19] = fma(kD, v[19], kE * v[15]);
      const double t2 = kG * ((v[11] + v[16]) + v[18]);
      w[11] = fma(kF, v[11], t2);
      w[16] = fma(kF, v[16], t2);
      w[18] = fma(kF, v[18], t2);
      w[21] = kH * v[21];
      w[22] = kH * v[22];
      w[23] = kH * v[23];
    }
    double T[3][4];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      T[c][0] = carry[c][0] + w[12 + c];
      carry[c][0] = -w[12 + c];
#pragma unroll
      for (int m = 1; m < 4; ++m) {
        T[c][m] = carry[c][m] + (w[3 * m + c] + w[3 * (m + 4) + c]);
        carry[c][m] = w[3 * m + c] - w[3 * (m + 4) + c];
      }
    }
    // stage node plane ek+2 into the buffer plane ek held (its last reader,
    // layer ek-1, is behind the previous barrier)
    if (ek + 1 < k1) {
      store_plane(cur ^ 1);
      load_plane(ek + 3);
    }
    if (ek < k0) {
      __syncthreads();
      return;
    }
    // xy inverse -> corner partials on plane ek; publish what the left,
    // lower and lower-left owners need
    double n11[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double S0 = T[c][0] + T[c][2], D0 = T[c][1] + T[c][3];
      const double S1 = T[c][0] - T[c][2], D1 = T[c][1] - T[c][3];
      pub[(pb * 9 + c) * nt + t] = S0 + D0;      // (y0, x0)
      pub[(pb * 9 + 3 + c) * nt + t] = S0 - D0;  // (y0, x1)
      pub[(pb * 9 + 6 + c) * nt + t] = S1 + D1;  // (y1, x0)
      n11[c] = S1 - D1;                          // (y1, x1)
    }
    __syncthreads();
    if (ek > k0) flush(pb ^ 1, ek - 1);  // plane ek-1's outputs, staged last layer
    if (own) {
      const double* pr = pub + pb * 9 * nt;
      const int64_t mnode = onode + int64_t(ek) * NX * NY;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        // (own (y1,x1) + right (y1,x0)) + (up (y0,x1) + up-right (y0,x0))
        const double lo = n11[c] + pr[(6 + c) * nt + t + 1];
        const double hi = pr[(3 + c) * nt + t + W] + pr[c * nt + t + W + 1];
        const bool fixed = g.xface ? oi == 0 : ((nmask[mnode] >> c) & 1);
        ost[pb * OL + oidx + c] = fixed ? 0.0 : lo + hi;
      }
    }
    pb ^= 1;
  };

  for (int ek = k0 - 1; ek < k1; ek += 2) {
    layer(ek, QA, QB);
    if (ek + 1 >= k1) break;
    layer(ek + 1, QB, QA);
  }
  __syncthreads();
  flush(pb ^ 1, k1 - 1);
}

// Tiling of the FP64 apply: T x tiles of W element columns (W - 1 owned node
// columns, NX split evenly), R rows (R - 1 owned node rows) with W*R <= 512,
// z chunks minimising waves x (chunk + 1 recomputed layer) on nsm SMs.
struct P64Plan {
  int W = 0, R = 0, tx = 0, ty = 0, kchunk = 0, nch = 0;
};
static P64Plan p64_plan(const GridDesc& g, int nsm, int maxt = kP64MaxThreads) {
  const int NX = g.nx + 1, NY = g.ny + 1, planes = g.nz + 1;
  nsm *= kP64MaxThreads / maxt;  // resident CTAs per wave
  P64Plan best;
  double best_cost = 1e300;
  for (int T = 1; T <= 16; ++T) {
    const int own_x = (NX + T - 1) / T;
    const int W = own_x + 1;
    if (W > maxt / 2 || own_x < std::min(NX, 15)) continue;
    const int R = std::min(maxt / W, NY + 1);
    if (R < 2) continue;
    const int ty = (NY + R - 2) / (R - 1);
    const int tiles = T * ty;
    const int threads = (W * R + 31) / 32 * 32;
    for (int c = 1; c <= planes; ++c) {
      const int kc = (planes + c - 1) / c;
      const int n = (planes + kc - 1) / kc;
      const long waves = (long(tiles) * n + nsm - 1) / nsm;
      const double cost = double(waves) * (kc + 1) * threads;
      if (cost < best_cost) {
        best_cost = cost;
        best.W = W;
        best.R = R;
        best.tx = T;
        best.ty = ty;
        best.kchunk = kc;
        best.nch = n;
      }
    }
  }
  return best;
}

bool p64_supported(const FineOp& op) {
  PkCoefD C;
  return op.walsh_ok && pk64_params(op, C);
}

void fine_apply_p64(const FineOp& op, const double* u, double* y, cudaStream_t s) {
  PkCoefD C;
  SG_REQUIRE(op.walsh_ok && pk64_params(op, C), "FP64 apply: element matrix lacks the Walsh block form");
  const GridDesc& g = op.grid.d;
  // 256-thread blocks, two independent CTAs per SM (still 16 warps at 128
  // registers; one CTA's FP64 dependency waits and per-layer barrier overlap
  // the other's work) at the price
  // of a taller y halo: 35.6 -> 35.0 us at 100^3, 211.7 -> 204 us at 200^3,
  // same bits (the owner sum order does not depend on the tiling).
  // SG_P64_NT=512 restores one 512-thread CTA per SM (A/B switch, read once).
  static const int nt_env = [] {
    const char* e = std::getenv("SG_P64_NT");
    return e && std::atoi(e) == 512 ? kP64MaxThreads : 256;
  }();
  P64Plan pl = p64_plan(g, num_sms(), nt_env);
  int threads = nt_env;
  if (pl.W == 0 && threads == 256) {  // rows too long for 256-thread tiles (NX > ~2000)
    threads = kP64MaxThreads;
    pl = p64_plan(g, num_sms(), threads);
  }
  SG_REQUIRE(pl.W > 0, "FP64 apply: no tiling for this grid");
  // always a full block (W * R <= block size; the extra threads only help
  // stage planes): the block size is then a compile-time constant of the
  // kernel (constant shared-memory offsets: 36.9 -> 35.3 us at 100^3)
  const int SL = (pl.R + 1) * 3 * (pl.W + 1);
  const size_t smem = sizeof(double) * (2 * size_t(SL) + 18 * size_t(threads) +
                                        2 * size_t(pl.R - 1) * 3 * (pl.W - 1));
  const int ld = (SL + threads - 1) / threads;
  dim3 grid(pl.tx, pl.ty, pl.nch);
  auto go = [&](auto kern) {
    static int attr = 0;
    if (attr < int(smem)) {
      SG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      attr = int(smem);
    }
    kern<<<grid, threads, smem, s>>>(g, op.grid.nmask.p, u, y, op.E64.p, C, pl.W, pl.R, pl.kchunk);
  };
  static const bool rt_nt = std::getenv("SG_P64_RTNT") != nullptr;
  static_assert(kP64MaxThreads == 512, "fine_p64_kernel<LD, 512> below");
  if (threads == 256 && ld <= 4) go(fine_p64_kernel<4, 256>);
  else if (threads == 256 && ld <= 8) go(fine_p64_kernel<8, 256>);
  else if (ld <= 4 && !rt_nt) go(fine_p64_kernel<4, 512>);
  else if (ld <= 4) go(fine_p64_kernel<4, 0>);
  else if (ld <= 6) go(fine_p64_kernel<6, 0>);
  else go(fine_p64_kernel<8, 0>);
  SG_REQUIRE(ld <= 8, "FP64 apply: slab too large for the tile");
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    throw Error(std::string("FP64 apply launch (") + std::to_string(pl.tx) + "," +
                std::to_string(pl.ty) + "," + std::to_string(pl.nch) + ")x" + std::to_string(threads) +
                " smem " + std::to_string(smem) + ": " + cudaGetErrorString(e));
  SG_CHECK_LAUNCH();
}

}  // namespace sg
