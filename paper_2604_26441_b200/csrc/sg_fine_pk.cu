// Level-0 matrix-free FP32 apply on packed FP32x2 arithmetic (FADD2 / FMUL2 /
// FFMA2, sm_100a).  fine_operator.py:56-77 (FP32 tag): y = K_ff u with the
// element modulus applied per element.
//
// Same algebra as sg_fine_walsh.cu (tensor Walsh basis, 45-entry Kw, SURVEY
// A.6) but re-tiled so that every FP32 instruction does two elements' work:
//  * a thread owns an x-PAIR of elements (e0, e1) = (ex, ex+1) of one element
//    row and streams the pair up a z-chunk; every Walsh, scaling, Kw and
//    inverse step runs on float2 lanes (e0, e1) -> half the FP32 issue slots;
//  * the separable transform is shared: the x/y stage of a node plane is
//    computed once and reused by the layer below and the layer above (in
//    registers); the inverse adds the two layers sharing a node plane in the
//    Walsh-xy domain before the xy inverse (12 adds instead of 24);
//  * a CTA = R element rows x P pairs, flattened (t = row*P + pair), so the
//    tile fits any nx (P = (nx+2)/2 pairs covers a whole row for nx <= 100 with
//    two phantom columns); neighbour partial sums go through shared memory
//    (one barrier per layer, double-buffered) in a fixed order, so every
//    output is bit-reproducible run to run;
//  * ownership: pair p owns node columns ex+1 and ex+2 (the last pair only
//    ex+1), local row r < R-1 owns node row ej+1; tiles overlap by one element
//    column / row / layer (recomputed halo, no atomics).
#include <cmath>
#include "sg_kernels.cuh"

namespace sg {


constexpr int kPkMaxThreads = 512;

__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  return __fadd2_rn(a, make_float2(-b.x, -b.y));
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
// A product that feeds an addition: two scalar mul.rn.f32.  ptxas contracts
// mul.rn.f32x2 followed by add.rn.f32x2 into FFMA2 (the .rn does not stop it
// for the packed forms), and it decides that per code copy: the same source
// then rounded differently in an unrolled copy or another instantiation.
// Scalar mul.rn is never contracted, so every rounding is the one written here.
__device__ __forceinline__ float2 mul2s(float2 a, float2 b) {
  return make_float2(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y));
}
// x/y stage of one node plane for an element pair: raw[y][x][c] (x = node
// columns ex, ex+1, ex+2; y = rows ej, ej+1) -> Q[c][m], m = mode in the xy
// Walsh basis (0: const, 1: x, 2: y, 3: xy), lanes = (e0, e1).
__device__ __forceinline__ void plane_xy(const float (&raw)[2][3][3], float2 (&Q)[3][4]) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    float2 S[2], D[2];
#pragma unroll
    for (int y = 0; y < 2; ++y) {
      const float2 A = make_float2(raw[y][0][c], raw[y][1][c]);  // x = 0 corners
      const float2 B = make_float2(raw[y][1][c], raw[y][2][c]);  // x = 1 corners
      S[y] = add2(A, B);
      D[y] = sub2(A, B);
    }
    Q[c][0] = add2(S[0], S[1]);
    Q[c][2] = sub2(S[0], S[1]);
    Q[c][1] = add2(D[0], D[1]);
    Q[c][3] = sub2(D[0], D[1]);
  }
}

// Block structure of Kw/64 (verified on the host by pk_params): with index
// 3*mode + comp the 45 nonzeros form
//   {3,7,14} and {11,16,18}: [[p,q,q],[q,p,q],[q,q,p]]  -> (p-q) v_i + q * sum
//   {4,6}, {5,12}, {8,13}:     [[c,c],[c,c]]            -> c * (v_i + v_j), both rows
//   {9,20}, {10,17}, {15,19}:  [[d,e],[e,d]]
//   {21}, {22}, {23}:          h
// so w = Kw (E v) costs 33 packed ops plus 8 per-element coefficient scalings
// (E folded into the coefficients) instead of 21 + 45.
struct PkCoef {
  float amb, b, c, d, e, fmg, g, h;
};

// Level-0 FP32 vectors in the "P32" layout: component-planar rows,
//   index(c, i, j, k) = ((k*NY + j)*3 + c)*XS + i,  XS = NX rounded up to even,
// padding (i >= NX) held at 0.  A pair's two x-nodes are one aligned 8-byte
// load/store and a warp's lanes touch contiguous 256 B: the node layout's
// 12-byte node stride made every scalar access span six 128-byte lines.
enum PkMode : int { PK_Y = 0, PK_CHEB = 1, PK_RES = 2 };

// Fused epilogues (smoothers.py:90-110 / hierarchy.py:214 rounding points,
// FP32 ops per lane, no contraction):
//  PK_CHEB: r = b - Kx; d' = A*(dinv*r) + AC*d (first: d' = A*(dinv*r));
//           x' = x + d'   (x' into a different buffer: neighbours still read x)
//  PK_RES:  out64 = r64 - f64(Kx)   (node layout FP64, the coarse-level residual)
struct PkEpi {
  const float* b = nullptr;
  const float* dinv = nullptr;
  float* d = nullptr;
  float* xout = nullptr;
  float A = 0.f, AC = 0.f;
  int first = 0;
  const double* r64 = nullptr;
  double* out64 = nullptr;
};

// Prefetch loads as volatile asm: issued where written (the compiler may not
// sink them next to their use to save registers, which exposed the latency).
__device__ __forceinline__ float ldp(const float* p) {
  float v;
  asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float2 ldp2(const float* p) {
  float2 v;
  asm volatile("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}

// XSC > 0: the row stride is the compile-time constant XSC (P32 rows padded to
// a multiple of 32 floats), so every address is base + immediate and the
// per-layer address arithmetic (IMAD on the FMA pipe) disappears; XSC = 0:
// runtime stride (rows wider than 256 nodes).
// NT: block size (512: one CTA per SM, 16 warps; 256: two CTAs per SM, so one
// CTA's per-layer barrier and epilogue overlap the other's transforms)
template <int MODE, int XSC, int NT>
__global__ void __launch_bounds__(NT, kPkMaxThreads / NT)
fine_pk_kernel(GridDesc g, const uint8_t* __restrict__ nmask, const float* __restrict__ u,
               float* __restrict__ yout, const float* __restrict__ E, PkCoef C, int P, int R,
               int kchunk, int XS_, int SX, PkEpi ep) {
  const int XS = XSC > 0 ? XSC : XS_;
  // published partials [buf][q][thread]: q 0..2 = i0(row 0), 3..5 = i1(row 0),
  // 6..8 = i2(row 0), 9..11 = i2(row 1), 3 comps each
  __shared__ float pub[2][12][NT];
  // PK_CHEB: this plane's b, dinv, x, d of the owned node pair, prefetched
  // with cp.async at the top of the layer ([q][thread], q = array*3 + comp)
  extern __shared__ float2 epre[];
  const int t = threadIdx.x, lane = t & 31;
  const int row = t / P, pair = t - row * P;
  const bool live = row < R;
  const int NX = g.nx + 1, NY = g.ny + 1;
  // x tiles (nx+1 > 128 nodes): tile t starts at node xo = t*SX (even) and
  // owns nodes [own_lo, own_hi); its first pair (no left neighbour) and last
  // pair are halo pairs except at the domain ends
  const int xo = int(blockIdx.x) * SX;
  const int own_lo = blockIdx.x == 0 ? 0 : xo + 2;
  const int own_hi = int(blockIdx.x) == int(gridDim.x) - 1 ? g.nx + 1 : xo + 2 * P - 2;
  const int ex = xo + 2 * pair;  // e0; nodes ex, ex+1, ex+2
  const int exl = min(ex, XS - 2);  // load column (phantom pairs past the row end read finite data)
  const int ej = int(blockIdx.y) * (R - 1) - 1 + row;
  const int k0 = int(blockIdx.z) * kchunk;
  const int k1 = min(k0 + kchunk, g.nz + 1);  // output node planes [k0, k1)
  const int64_t pl = int64_t(3) * XS * NY;    // one node plane in P32
  // i2 comes from lane+1's first node unless lane+1 is another row / warp
  const bool fix = lane == 31 || pair == P - 1 || !live;
  // row pointers (rows ej, ej+1, clamped), one node plane per layer
  const float* up[2];
  {
    const int pk = min(max(k0 - 1, 0), g.nz);
#pragma unroll
    for (int y = 0; y < 2; ++y)
      up[y] = u + int64_t(pk) * pl + int64_t(3) * XS * min(max(ej + y, 0), g.ny) + exl;
  }
  const bool rowin = live && ej >= 0 && ej < g.ny;
  const float m0 = (rowin && ex < g.nx) ? 1.f : 0.f;
  const float m1 = (rowin && ex + 1 < g.nx) ? 1.f : 0.f;
  const int64_t estride = int64_t(g.nx) * g.ny;
  const int64_t erow = int64_t(g.nx) * min(max(ej, 0), g.ny - 1);
  const float* Ep0 = E + erow + min(ex, g.nx - 1);
  const float* Ep1 = E + erow + min(ex + 1, g.nx - 1);

  // ownership: nodes (ex, ex+1) of node row ej+1
  const int on = ej + 1;
  const bool own = live && row < R - 1 && on >= 0 && on <= g.ny && ex >= own_lo && ex < own_hi;
  const bool own1 = ex + 1 < own_hi;
  const int64_t orow = int64_t(3) * XS * max(on, 0) + ex + int64_t(k0) * pl;  // + c*XS
  const int64_t onode = int64_t(ex) + int64_t(NX) * max(on, 0) + int64_t(k0) * NX * NY;

  float2 Qlo[3][4], Qhi[3][4], carry[3][4];
  float2 A[2][3];
  float a2[2][3];
  auto load_plane = [&]() {
#pragma unroll
    for (int y = 0; y < 2; ++y)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        A[y][c] = ldp2(up[y] + c * XS);
        a2[y][c] = ldp(up[y] + c * XS + (fix && exl + 2 < XS ? 2 : 0));
      }
  };
  auto plane_q = [&](float2 (&Q)[3][4]) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      float2 S[2], D[2];
#pragma unroll
      for (int y = 0; y < 2; ++y) {
        const float nb = __shfl_down_sync(0xffffffffu, A[y][c].x, 1);
        const float2 B = make_float2(A[y][c].y, fix ? a2[y][c] : nb);
        S[y] = add2(A[y][c], B);
        D[y] = sub2(A[y][c], B);
      }
      Q[c][0] = add2(S[0], S[1]);
      Q[c][2] = sub2(S[0], S[1]);
      Q[c][1] = add2(D[0], D[1]);
      Q[c][3] = sub2(D[0], D[1]);
    }
  };
  auto advance = [&](bool more) {
    if (more) {
      up[0] += pl;
      up[1] += pl;
    }
  };
  int pk = k0 - 1;
  load_plane();
  plane_q(Qlo);
  advance(pk >= 0 && pk < g.nz);
  ++pk;
  load_plane();  // plane k0
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int m = 0; m < 4; ++m) carry[c][m] = make_float2(0.f, 0.f);
  int buf = 0;
  int64_t oplane = 0;  // output planes written so far
  // element moduli, prefetched one layer ahead (0 outside the domain)
  // raw moduli of layer ek (the domain mask is applied when they are used)
  auto load_E = [&](int ek) {
    const int64_t eo = int64_t(min(max(ek, 0), g.nz - 1)) * estride;
    return make_float2(ldp(Ep0 + eo), ldp(Ep1 + eo));
  };
  float2 Eraw = load_E(k0 - 1);

  // plain apply: two layers per trip, so the plane transforms alternate
  // between Qlo and Qhi without register copies (safe for the bits because no
  // product is contracted, mul2s above); the fused modes spill when unrolled
#pragma unroll(MODE == PK_Y ? 2 : 1)
  for (int ek = k0 - 1; ek < k1; ++ek) {
    plane_q(Qhi);  // node plane ek+1
    advance(pk >= 0 && pk < g.nz);
    ++pk;
    load_plane();  // prefetch node plane ek+2
    if constexpr (MODE == PK_CHEB) {
      if (ek >= k0 && own) {
        const float* src[4] = {ep.b, ep.dinv, u, ep.d};
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const unsigned dst = static_cast<unsigned>(
                __cvta_generic_to_shared(epre + (a * 3 + c) * NT + t));
            const float* gp = src[a] + orow + oplane * pl + int64_t(c) * XS;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(gp) : "memory");
          }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    const float2 En = load_E(ek + 1);
    const bool kin = ek >= 0 && ek < g.nz;
    const float2 Es = mul2(Eraw, make_float2(kin ? m0 : 0.f, kin ? m1 : 0.f));
    const float2 kA = mul2(Es, make_float2(C.amb, C.amb)), kB = mul2(Es, make_float2(C.b, C.b));
    const float2 kC = mul2(Es, make_float2(C.c, C.c)), kD = mul2(Es, make_float2(C.d, C.d));
    const float2 kE = mul2(Es, make_float2(C.e, C.e)), kF = mul2(Es, make_float2(C.fmg, C.fmg));
    const float2 kG = mul2(Es, make_float2(C.g, C.g)), kH = mul2(Es, make_float2(C.h, C.h));
    // z stage -> v[3*mode + c], modes 1..7
    float2 v[24];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
#pragma unroll
      for (int m = 1; m < 4; ++m) v[3 * m + c] = add2(Qlo[c][m], Qhi[c][m]);
#pragma unroll
      for (int m = 0; m < 4; ++m) v[3 * (m + 4) + c] = sub2(Qlo[c][m], Qhi[c][m]);
    }
    // w = (E Kw) v, block form
    float2 w[24];
    {
      const float2 t1 = mul2(kB, add2(add2(v[3], v[7]), v[14]));
      w[3] = fma2(kA, v[3], t1);
      w[7] = fma2(kA, v[7], t1);
      w[14] = fma2(kA, v[14], t1);
      w[4] = w[6] = mul2s(kC, add2(v[4], v[6]));
      w[5] = w[12] = mul2s(kC, add2(v[5], v[12]));
      w[8] = w[13] = mul2s(kC, add2(v[8], v[13]));
      w[9] = fma2(kD, v[9], mul2(kE, v[20]));
      w[20] = fma2(kD, v[20], mul2(kE, v[9]));
      w[10] = fma2(kD, v[10], mul2(kE, v[17]));
      w[17] = fma2(kD, v[17], mul2(kE, v[10]));
      w[15] = fma2(kD, v[15], mul2(kE, v[19]));
      w[19] = fma2(kD, v[19], mul2(kE, v[15]));
      const float2 t2 = mul2(kG, add2(add2(v[11], v[16]), v[18]));
      w[11] = fma2(kF, v[11], t2);
      w[16] = fma2(kF, v[16], t2);
      w[18] = fma2(kF, v[18], t2);
      w[21] = mul2s(kH, v[21]);
      w[22] = mul2s(kH, v[22]);
      w[23] = mul2s(kH, v[23]);
    }
    // inverse z stage + the layer below's top half (same node plane ek)
    float2 T[3][4];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      T[c][0] = add2(carry[c][0], w[12 + c]);
      carry[c][0] = make_float2(-w[12 + c].x, -w[12 + c].y);
#pragma unroll
      for (int m = 1; m < 4; ++m) {
        T[c][m] = add2(carry[c][m], add2(w[3 * m + c], w[3 * (m + 4) + c]));
        carry[c][m] = sub2(w[3 * m + c], w[3 * (m + 4) + c]);
      }
    }
    if (ek >= k0) {
      // xy inverse -> corner partials of this pair on plane ek
      float n0[2][3], n1[2][3], n2[2][3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float2 S0 = add2(T[c][0], T[c][2]), D0 = add2(T[c][1], T[c][3]);
        const float2 S1 = sub2(T[c][0], T[c][2]), D1 = sub2(T[c][1], T[c][3]);
        const float2 r0x0 = add2(S0, D0), r0x1 = sub2(S0, D0);
        const float2 r1x0 = add2(S1, D1), r1x1 = sub2(S1, D1);
        n0[0][c] = r0x0.x;
        n1[0][c] = r0x1.x + r0x0.y;
        n2[0][c] = r0x1.y;
        n0[1][c] = r1x0.x;
        n1[1][c] = r1x1.x + r1x0.y;
        n2[1][c] = r1x1.y;
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        pub[buf][c][t] = n0[0][c];
        pub[buf][3 + c][t] = n1[0][c];
        pub[buf][6 + c][t] = n2[0][c];
        pub[buf][9 + c][t] = n2[1][c];
      }
      if constexpr (MODE == PK_CHEB) asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();
      if (own) {
        const bool left = pair > 0;
        const int64_t nodei = onode + oplane * int64_t(NX) * NY;
        float yr[2][3];  // PK_RES: the pair's 6 values, written together below
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          // node ex: (own e0 + left pair's e1) + (same, row above)
          float y0 = n0[1][c] + (left ? pub[buf][9 + c][t - 1] : 0.f);
          y0 = y0 + (pub[buf][c][t + P] + (left ? pub[buf][6 + c][t + P - 1] : 0.f));
          // node ex+1: own pair + the row above's pair
          float y1 = n1[1][c] + pub[buf][3 + c][t + P];
          const bool f0 = g.xface ? ex == 0 : ((nmask[nodei] >> c) & 1);
          const bool f1 = !own1 || (g.xface ? false : ((nmask[nodei + 1] >> c) & 1));
          y0 = f0 ? 0.f : y0;
          y1 = f1 ? 0.f : y1;
          const int64_t o = orow + oplane * pl + int64_t(c) * XS;
          if constexpr (MODE == PK_Y) {
            *reinterpret_cast<float2*>(yout + o) = make_float2(y0, y1);
          } else if constexpr (MODE == PK_CHEB) {
            const float2 bb = epre[(0 + c) * NT + t];
            const float2 di = epre[(3 + c) * NT + t];
            const float2 xx = epre[(6 + c) * NT + t];
            // scalar round-to-nearest intrinsics: never contracted (ptxas
            // was seen fusing even explicit mul.rn/add.rn .f32x2 into FFMA2)
            float2 dn = make_float2(__fmul_rn(ep.A, __fmul_rn(di.x, __fsub_rn(bb.x, y0))),
                                    __fmul_rn(ep.A, __fmul_rn(di.y, __fsub_rn(bb.y, y1))));
            if (!ep.first) {
              const float2 dd = epre[(9 + c) * NT + t];
              dn.x = __fadd_rn(dn.x, __fmul_rn(ep.AC, dd.x));
              dn.y = __fadd_rn(dn.y, __fmul_rn(ep.AC, dd.y));
            }
            *reinterpret_cast<float2*>(ep.d + o) = dn;
            const float2 xn = make_float2(__fadd_rn(xx.x, dn.x), __fadd_rn(xx.y, dn.y));
            *reinterpret_cast<float2*>(ep.xout + o) = xn;
            yr[0][c] = xn.x;  // last smoothing step: the f64 node-layout iterate (below)
            yr[1][c] = xn.y;
          } else {
            yr[0][c] = y0;
            yr[1][c] = y1;
          }
        }
        if constexpr (MODE == PK_CHEB) {
          if (ep.out64) {  // 6 contiguous doubles: 16-byte stores where aligned
            const int64_t q = 3 * nodei;
            double* op = ep.out64 + q;
            if (own1) {
              double ov[6];
#pragma unroll
              for (int k = 0; k < 6; ++k) ov[k] = double(yr[k / 3][k % 3]);
              if ((q & 1) == 0) {
#pragma unroll
                for (int k = 0; k < 3; ++k)
                  *reinterpret_cast<double2*>(op + 2 * k) = make_double2(ov[2 * k], ov[2 * k + 1]);
              } else {
                op[0] = ov[0];
                *reinterpret_cast<double2*>(op + 1) = make_double2(ov[1], ov[2]);
                *reinterpret_cast<double2*>(op + 3) = make_double2(ov[3], ov[4]);
                op[5] = ov[5];
              }
            } else {
#pragma unroll
              for (int c = 0; c < 3; ++c) op[c] = double(yr[0][c]);
            }
          }
        }
        if constexpr (MODE == PK_RES) {
          // nodes ex, ex+1 are 6 contiguous doubles in the node layout: 16-byte
          // accesses (8 + 16 + 16 + 8 when the pair starts on an odd double)
          // instead of six 24-byte-strided ones; same arithmetic, same bits
          const int64_t q = 3 * nodei;
          const double* rp = ep.r64 + q;
          double* op = ep.out64 + q;
          if (own1) {
            double rv[6];
            if ((q & 1) == 0) {
#pragma unroll
              for (int k = 0; k < 3; ++k) {
                const double2 v = *reinterpret_cast<const double2*>(rp + 2 * k);
                rv[2 * k] = v.x;
                rv[2 * k + 1] = v.y;
              }
            } else {
              rv[0] = rp[0];
              const double2 a = *reinterpret_cast<const double2*>(rp + 1);
              const double2 b = *reinterpret_cast<const double2*>(rp + 3);
              rv[1] = a.x; rv[2] = a.y; rv[3] = b.x; rv[4] = b.y;
              rv[5] = rp[5];
            }
            double ov[6];
#pragma unroll
            for (int k = 0; k < 6; ++k) ov[k] = __dsub_rn(rv[k], double(yr[k / 3][k % 3]));
            if ((q & 1) == 0) {
#pragma unroll
              for (int k = 0; k < 3; ++k)
                *reinterpret_cast<double2*>(op + 2 * k) = make_double2(ov[2 * k], ov[2 * k + 1]);
            } else {
              op[0] = ov[0];
              *reinterpret_cast<double2*>(op + 1) = make_double2(ov[1], ov[2]);
              *reinterpret_cast<double2*>(op + 3) = make_double2(ov[3], ov[4]);
              op[5] = ov[5];
            }
          } else {
#pragma unroll
            for (int c = 0; c < 3; ++c) op[c] = __dsub_rn(rp[c], double(yr[0][c]));
          }
        }
      }
      ++oplane;
      buf ^= 1;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int m = 0; m < 4; ++m) Qlo[c][m] = Qhi[c][m];
    Eraw = En;
  }
}

// Block parameters of Kw/64 (fp32); false when Ke does not have the block
// structure (the scalar Walsh kernel is used instead).
static bool pk_params(const FineOp& op, PkCoef& C) {
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
  C.amb = float(a - b);
  C.b = float(b);
  C.c = float(c);
  C.d = float(d);
  C.e = float(e);
  C.fmg = float(f - gg);
  C.g = float(gg);
  C.h = float(h);
  return true;
}

// Row stride of the P32 layout: NX rounded up to a multiple of 32 floats up to
// 256 (compile-time strides for the apply kernel), else to even.
int p32_xs(const GridDesc& g) {
  const int nx1 = g.nx + 1;
  return nx1 <= 256 ? (nx1 + 31) & ~31 : (nx1 + 1) & ~1;
}
int64_t p32_size(const GridDesc& g) {
  return int64_t(3) * p32_xs(g) * (g.ny + 1) * (g.nz + 1) + 4;  // + slack for the i2 reads
}

bool p32_supported(const FineOp& op) {
  PkCoef C;
  return op.walsh_ok && pk_params(op, C);
}

// Work plan of the P32 kernel (host only; sg_plan_p32 exposes it for tests).
// x: one tile per row when (nx+2)/2 <= 64 pairs, else T tiles of P pairs
// overlapping by two pairs (stride SX = 2P - 4 nodes), P as small as T
// allows; y: tiles of R element rows overlapping by one; z: chunks of kchunk
// node planes (+ one recomputed layer) minimising waves x (chunk + 1).
// Block size of the P32 kernels.  512 threads = one CTA (16 warps) per SM;
// 256 = two CTAs per SM, each CTA's per-layer barrier and epilogue then
// overlapping the other's transforms, at the price of a taller y halo (R - 1
// of R rows owned).  Measured at 100^3 (bit-identical): the fused smoother
// 33.6 -> 31.4 us and the fused residual 31.0 -> 30.0 us at 256, the plain
// apply 22.3 -> 22.8 us; at 200^3 (R = 4 at 256) every mode is slower.  So
// the fused modes run 256-thread blocks when that still leaves R >= 5 rows.
// SG_PK_NT=256|512 forces one size for every mode (A/B switch, read once).
int pk_threads(const GridDesc& g, int mode) {
  static const int env = [] {
    const char* e = getenv("SG_PK_NT");
    const int v = e ? atoi(e) : 0;
    return v == 256 || v == 512 ? v : 0;
  }();
  if (env) return env;
  const int P = (g.nx + 2) / 2;
  return mode != PK_Y && P <= 64 && 256 / P >= 5 ? 256 : kPkMaxThreads;
}

PkPlan pk_plan(const GridDesc& g, int nsm, int nt) {
  PkPlan pl;
  nsm *= kPkMaxThreads / nt;  // resident CTAs per wave
  int P = (g.nx + 2) / 2, T = 1, SX = 2 * P;
  if (P > 64) {
    for (T = 2;; ++T) {
      P = (g.nx + 1 + 4 * (T - 1) + 2 * T - 1) / (2 * T);
      if (P <= 64) break;
    }
    SX = 2 * P - 4;
  }
  int R = std::max(2, nt / P);
  R = std::min(R, g.ny + 2);
  const int tilesy = (g.ny + 1 + (R - 1) - 1) / (R - 1);
  const int planes = g.nz + 1;
  const int tiles = T * tilesy;
  int nch = 1;
  long best = 1L << 60;
  for (int c = 1; c <= planes; ++c) {
    const int kc = (planes + c - 1) / c;
    const int n = (planes + kc - 1) / kc;
    const long waves = (long(tiles) * n + nsm - 1) / nsm;
    const long cost = waves * (kc + 1);
    if (cost < best) { best = cost; nch = n; }
  }
  const int kchunk = (planes + nch - 1) / nch;
  nch = (planes + kchunk - 1) / kchunk;
  pl.P = P; pl.T = T; pl.SX = SX; pl.R = R; pl.tilesy = tilesy; pl.kchunk = kchunk; pl.nch = nch;
  pl.nt = nt;
  return pl;
}

template <int MODE>
static void launch_pk(const FineOp& op, const float* u, float* y, const PkEpi& ep, cudaStream_t s) {
  PkCoef C;
  SG_REQUIRE(op.walsh_ok && pk_params(op, C), "P32 apply: element matrix lacks the Walsh block form");
  const GridDesc& g = op.grid.d;
  const PkPlan pl = pk_plan(g, num_sms(), pk_threads(g, MODE));
  const int P = pl.P, R = pl.R, SX = pl.SX, kchunk = pl.kchunk;
  const int threads = ((P * R + 31) / 32) * 32;
  dim3 grid(pl.T, pl.tilesy, pl.nch);
  const int XS = p32_xs(g);
  static bool attr_set[2][9] = {};
  auto go = [&](auto kern, auto ntc) {
    constexpr int NT = decltype(ntc)::value;
    const size_t dyn = MODE == PK_CHEB ? sizeof(float2) * 12 * NT : 0;
    const int slot = XS <= 256 && XS % 32 == 0 ? XS / 32 : 0;
    if (MODE == PK_CHEB && !attr_set[NT == 256][slot]) {
      SG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn)));
      attr_set[NT == 256][slot] = true;
    }
    kern<<<grid, threads, dyn, s>>>(g, op.grid.nmask.p, u, y, op.E32.p, C, P, R, kchunk, XS, SX, ep);
  };
  auto by_xs = [&](auto ntc) {
    constexpr int NT = decltype(ntc)::value;
    // (the fused Chebyshev variant keeps the runtime stride: with a constant one
    // ptxas hoists more offsets and spills; measured slower)
    switch (MODE == PK_CHEB ? 0 : XS) {
      case 32: go(fine_pk_kernel<MODE, 32, NT>, ntc); break;
      case 64: go(fine_pk_kernel<MODE, 64, NT>, ntc); break;
      case 96: go(fine_pk_kernel<MODE, 96, NT>, ntc); break;
      case 128: go(fine_pk_kernel<MODE, 128, NT>, ntc); break;
      case 160: go(fine_pk_kernel<MODE, 160, NT>, ntc); break;
      case 192: go(fine_pk_kernel<MODE, 192, NT>, ntc); break;
      case 224: go(fine_pk_kernel<MODE, 224, NT>, ntc); break;
      case 256: go(fine_pk_kernel<MODE, 256, NT>, ntc); break;
      default: go(fine_pk_kernel<MODE, 0, NT>, ntc); break;
    }
  };
  if (pl.nt == 256) by_xs(std::integral_constant<int, 256>{});
  else by_xs(std::integral_constant<int, 512>{});
  SG_CHECK_LAUNCH();
}

void fine_apply_p32(const FineOp& op, const float* u, float* y, cudaStream_t s) {
  launch_pk<PK_Y>(op, u, y, PkEpi{}, s);
}
void fine_apply_p32_cheb(const FineOp& op, const float* x, float* xout, const float* b,
                         const float* dinv, float* d, float A, float AC, bool first, cudaStream_t s,
                         double* xout64) {
  PkEpi ep;
  ep.out64 = xout64;
  ep.b = b;
  ep.dinv = dinv;
  ep.d = d;
  ep.xout = xout;
  ep.A = A;
  ep.AC = AC;
  ep.first = first ? 1 : 0;
  launch_pk<PK_CHEB>(op, x, nullptr, ep, s);
}
void fine_apply_p32_res(const FineOp& op, const float* x, const double* r64, double* out64,
                        cudaStream_t s) {
  PkEpi ep;
  ep.r64 = r64;
  ep.out64 = out64;
  launch_pk<PK_RES>(op, x, nullptr, ep, s);
}

// chebyshev_smooth with x0=None on the P32 level (smoothers.py:90-99):
// b32 = f32(b64); d = c0*(dinv*b32); x = 0 + d -- one pass from the f64
// node-layout right-hand side.  A thread takes an x-pair of nodes: its six
// contiguous doubles in, one aligned float2 per component and array out
// (padding entries are never written: zero since allocation).
__global__ void cheb_first0_p32_kernel(GridDesc g, int XS, const double* __restrict__ b64,
                                       const float* __restrict__ dinv, float c0,
                                       float* __restrict__ b32, float* __restrict__ d,
                                       float* __restrict__ x, int npr, int64_t npairs) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= npairs) return;
  const int t32 = int(t);  // 32-bit index math (pairs < 2^31)
  const int jk = t32 / npr;
  const int i0 = 2 * (t32 - jk * npr);
  const bool two = i0 + 1 <= g.nx;
  const int64_t node = int64_t(jk) * (g.nx + 1) + i0;
  const double* bp = b64 + 3 * node;
  double bv[6];
#pragma unroll
  for (int k = 0; k < 3; ++k) bv[k] = bp[k];
#pragma unroll
  for (int k = 3; k < 6; ++k) bv[k] = two ? bp[k] : 0.0;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const int64_t q = (int64_t(jk) * 3 + c) * XS + i0;
    const float2 di = *reinterpret_cast<const float2*>(dinv + q);
    const float b0 = __double2float_rn(bv[c]), b1 = __double2float_rn(bv[3 + c]);
    const float d0 = __fmul_rn(c0, __fmul_rn(di.x, b0)), d1 = __fmul_rn(c0, __fmul_rn(di.y, b1));
    if (two) {
      *reinterpret_cast<float2*>(b32 + q) = make_float2(b0, b1);
      *reinterpret_cast<float2*>(d + q) = make_float2(d0, d1);
      *reinterpret_cast<float2*>(x + q) = make_float2(__fadd_rn(0.f, d0), __fadd_rn(0.f, d1));
    } else {
      b32[q] = b0;
      d[q] = d0;
      x[q] = __fadd_rn(0.f, d0);
    }
  }
}
void cheb_first0_p32(const GridDesc& g, const double* b64, const float* dinv, float c0, float* b32,
                     float* d, float* x, cudaStream_t s) {
  const int npr = (g.nx + 2) / 2;  // node pairs per row
  const int64_t npairs = int64_t(npr) * (g.ny + 1) * (g.nz + 1);
  cheb_first0_p32_kernel<<<grid_blocks(npairs, 256), 256, 0, s>>>(g, p32_xs(g), b64, dinv, c0, b32, d, x,
                                                                  npr, npairs);
  SG_CHECK_LAUNCH();
}

// ------------------------------------------------ P32 <-> node conversions
template <class Tin>
__global__ void to_p32_kernel(GridDesc g, int XS, const Tin* __restrict__ src, float* __restrict__ dst,
                              int64_t n) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int q32 = int(q);  // 32-bit index math (P32 vectors < 2^31 entries)
  const int rc = q32 / XS;
  const int i = q32 - rc * XS;  // (k*NY + j)*3 + c
  const int r3 = rc / 3, c = rc - 3 * r3;
  const int64_t node = int64_t(r3) * (g.nx + 1) + i;
  dst[q] = i <= g.nx ? float(src[3 * node + c]) : 0.f;
}
template <class Tout>
__global__ void from_p32_kernel(GridDesc g, int XS, const float* __restrict__ src, Tout* __restrict__ dst,
                                int64_t nd) {
  const int64_t d = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (d >= nd) return;
  const int d32 = int(d), node = d32 / 3, c = d32 - 3 * node;  // 32-bit index math
  const int jk = node / (g.nx + 1);
  const int i = node - jk * (g.nx + 1);
  dst[d] = Tout(src[(int64_t(jk) * 3 + c) * XS + i]);
}
template <class Tin>
void to_p32(const GridDesc& g, const Tin* src, float* dst, cudaStream_t s) {
  const int64_t n = int64_t(3) * p32_xs(g) * (g.ny + 1) * (g.nz + 1);
  to_p32_kernel<Tin><<<grid_blocks(n, 256), 256, 0, s>>>(g, p32_xs(g), src, dst, n);
  SG_CHECK_LAUNCH();
}
template <class Tout>
void from_p32(const GridDesc& g, const float* src, Tout* dst, cudaStream_t s) {
  const int64_t nd = 3 * g.nnodes();
  from_p32_kernel<Tout><<<grid_blocks(nd, 256), 256, 0, s>>>(g, p32_xs(g), src, dst, nd);
  SG_CHECK_LAUNCH();
}
template void to_p32<double>(const GridDesc&, const double*, float*, cudaStream_t);
template void to_p32<float>(const GridDesc&, const float*, float*, cudaStream_t);
template void from_p32<double>(const GridDesc&, const float*, double*, cudaStream_t);
template void from_p32<float>(const GridDesc&, const float*, float*, cudaStream_t);

}  // namespace sg
