// Hierarchy build and V/W-cycle (hierarchy.py:181-282), smoothers
// (smoothers.py:67-152), all device-resident.
//
// Rounding points mirror the reference: the smoother of a
// reduced-precision level runs its recurrence in FP32 with the coefficients
// rounded to FP32 (wt(1/sigma), wt(a), wt(a*c)); the residual handed to the
// coarse level is r64 - f64(K_tag x); transfers and coarse corrections are
// FP64.  Elementwise updates use explicit round-to-nearest intrinsics so no
// FMA contraction changes the numpy-equivalent bits.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include "sg_hier.cuh"

namespace sg {

template <class T> __device__ __forceinline__ T fmul(T a, T b);
template <> __device__ __forceinline__ double fmul<double>(double a, double b) { return __dmul_rn(a, b); }
template <> __device__ __forceinline__ float fmul<float>(float a, float b) { return __fmul_rn(a, b); }
template <class T> __device__ __forceinline__ T fadd(T a, T b);
template <> __device__ __forceinline__ double fadd<double>(double a, double b) { return __dadd_rn(a, b); }
template <> __device__ __forceinline__ float fadd<float>(float a, float b) { return __fadd_rn(a, b); }
template <class T> __device__ __forceinline__ T fsub(T a, T b);
template <> __device__ __forceinline__ double fsub<double>(double a, double b) { return __dsub_rn(a, b); }
template <> __device__ __forceinline__ float fsub<float>(float a, float b) { return __fsub_rn(a, b); }

#define SG_ELEMWISE(n) \
  const int64_t i_ = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; \
  if (i_ >= (n)) return;

// ---------------------------------------------------------- smoother kernels
// d = c0*(dinv*b); x = 0 + d   (chebyshev_smooth x0=None, smoothers.py:277-283)
template <class T>
__global__ void cheb_first0_kernel(int64_t n, const T* __restrict__ dinv, const T* __restrict__ b,
                                   T c0, T* __restrict__ d, T* __restrict__ x) {
  SG_ELEMWISE(n);
  const T dv = fmul(c0, fmul(dinv[i_], b[i_]));
  d[i_] = dv;
  x[i_] = fadd(T(0), dv);
}
// r = b - y; d = c0*(dinv*r); x = x + d
template <class T>
__global__ void cheb_first_kernel(int64_t n, const T* __restrict__ dinv, const T* __restrict__ b,
                                  const T* __restrict__ y, T c0, T* __restrict__ d, T* __restrict__ x) {
  SG_ELEMWISE(n);
  const T r = fsub(b[i_], y[i_]);
  const T dv = fmul(c0, fmul(dinv[i_], r));
  d[i_] = dv;
  x[i_] = fadd(x[i_], dv);
}
// r = b - y; d = A*(dinv*r) + AC*d; x = x + d   (smoothers.py:104-108)
template <class T>
__global__ void cheb_step_kernel(int64_t n, const T* __restrict__ dinv, const T* __restrict__ b,
                                 const T* __restrict__ y, T A, T AC, T* __restrict__ d, T* __restrict__ x) {
  SG_ELEMWISE(n);
  const T r = fsub(b[i_], y[i_]);
  const T dv = fadd(fmul(A, fmul(dinv[i_], r)), fmul(AC, d[i_]));
  d[i_] = dv;
  x[i_] = fadd(x[i_], dv);
}
// x = w*(dinv*b)   (jacobi_smooth x0=None)
template <class T>
__global__ void jac_first0_kernel(int64_t n, const T* __restrict__ dinv, const T* __restrict__ b, T w,
                                  T* __restrict__ x) {
  SG_ELEMWISE(n);
  x[i_] = fmul(w, fmul(dinv[i_], b[i_]));
}
// x = x + w*(dinv*(b - y))
template <class T>
__global__ void jac_step_kernel(int64_t n, const T* __restrict__ dinv, const T* __restrict__ b,
                                const T* __restrict__ y, T w, T* __restrict__ x) {
  SG_ELEMWISE(n);
  x[i_] = fadd(x[i_], fmul(w, fmul(dinv[i_], fsub(b[i_], y[i_]))));
}
// d64 = r - f64(y)
template <class T>
__global__ void residual_kernel(int64_t n, const double* __restrict__ r, const T* __restrict__ y,
                                double* __restrict__ d) {
  SG_ELEMWISE(n);
  d[i_] = __dsub_rn(r[i_], double(y[i_]));
}
__global__ void add_kernel(int64_t n, const double* __restrict__ a, double* __restrict__ x) {
  SG_ELEMWISE(n);
  x[i_] = __dadd_rn(x[i_], a[i_]);
}
__global__ void copy_kernel(int64_t n, const double* __restrict__ a, double* __restrict__ b) {
  SG_ELEMWISE(n);
  b[i_] = a[i_];
}
__global__ void recip_kernel(int64_t n, const double* __restrict__ d, double* __restrict__ di,
                             float* __restrict__ di32) {
  SG_ELEMWISE(n);
  const double v = d[i_] != 0.0 ? __drcp_rn(d[i_]) : 0.0;
  di[i_] = v;
  di32[i_] = __double2float_rn(v);
}

template <class K>
static void launch_ew(int64_t n, cudaStream_t s, K kernel_launch) {
  kernel_launch(grid_blocks(n, 256), 256);
  SG_CHECK_LAUNCH();
}

// ---------------------------------------------------------------- applies
void fine_apply_tag(const FineOp& op, int tag, const void* x, void* y, cudaStream_t s) {
  switch (tag) {
    case TAG_FP64: fine_apply_f64(op, (const double*)x, (double*)y, s); break;
    case TAG_FP32: fine_apply_f32(op, (const float*)x, (float*)y, s); break;
    case TAG_BF16: fine_apply_bf16(op, (const float*)x, (float*)y, s); break;
    default: throw Error("bad precision tag");
  }
}

void level_apply(Hier& H, Level& L, int tag, const void* x, void* y, cudaStream_t s) {
  if (H.comm) H.comm->exchange(L.idx, x, tag == TAG_FP64 ? 8 : 4, s);
  if (L.is_fine) {
    fine_apply_tag(*H.fine, tag, x, y, s);
    return;
  }
  if (tag == TAG_FP64 && L.st.T64s.p) {
    stencil_sym64(*L.g, L.st.T64s.p, 0, (const double*)x, (double*)y, nullptr, nullptr, nullptr, 0.0, 0.0,
                  true, s);
  } else if (tag == TAG_FP64) {
    stencil_apply<double>(*L.g, L.st.T64.p, (const double*)x, (double*)y, s);
  } else if (tag == TAG_FP32) {
    SG_REQUIRE(L.st.T32.p, "fp32 operator copy missing");
    stencil_apply<float>(*L.g, L.st.T32.p, (const float*)x, (float*)y, s);
  } else {
    throw Error("bf16 tag on an assembled level is not produced by any policy");
  }
}

// Working-type dispatch for the smoother.
template <class T>
struct WT;
template <>
struct WT<double> {
  static double* x(Level& L) { return L.w.x.p; }
  static double* y(Level& L) { return L.w.y64.p; }
  static double* d(Level& L) { return L.w.dd64.p; }
  static const double* dinv(Level& L) { return L.dinv.p; }
};
template <>
struct WT<float> {
  static float* x(Level& L) { return L.w.x32.p; }
  static float* y(Level& L) { return L.w.y32.p; }
  static float* d(Level& L) { return L.w.dd32.p; }
  static const float* dinv(Level& L) { return L.dinv32.p; }
};

template <class T>
static void smooth_t(Hier& H, Level& L, const T* b, const double* x0, double* out, cudaStream_t s) {
  const int64_t n = L.nd();
  T* x = WT<T>::x(L);
  T* y = WT<T>::y(L);
  T* d = WT<T>::d(L);
  const T* dinv = WT<T>::dinv(L);
  auto to_w = [&](const double* src) {
    if constexpr (sizeof(T) == 8) {
      if (src != (const double*)x) launch_ew(n, s, [&](int nb, int nt) { copy_kernel<<<nb, nt, 0, s>>>(n, src, (double*)x); });
    } else {
      cvt_f64_to_f32(n, src, (float*)x, s);
    }
  };
  if (L.kind == 0) {  // Chebyshev (smoothers.py:67-110)
    const double lam = L.lam;
    const double sigma = 0.5 * (lam + L.alpha * lam);
    const double delta = 0.5 * (lam - L.alpha * lam);
    const T c0 = T(1.0 / sigma);
    if (!x0) {
      launch_ew(n, s, [&](int nb, int nt) { cheb_first0_kernel<T><<<nb, nt, 0, s>>>(n, dinv, b, c0, d, x); });
    } else {
      to_w(x0);
      level_apply(H, L, L.tag, x, y, s);
      launch_ew(n, s, [&](int nb, int nt) { cheb_first_kernel<T><<<nb, nt, 0, s>>>(n, dinv, b, y, c0, d, x); });
    }
    double a = 2.0 / sigma;
    for (int it = 1; it < L.degree; ++it) {
      level_apply(H, L, L.tag, x, y, s);
      const double c = delta * delta * a / 4.0;
      a = 1.0 / (sigma - c);
      const T A = T(a), AC = T(a * c);
      launch_ew(n, s, [&](int nb, int nt) { cheb_step_kernel<T><<<nb, nt, 0, s>>>(n, dinv, b, y, A, AC, d, x); });
    }
  } else {  // damped Jacobi (smoothers.py:113-131)
    const T w = T(L.omega);
    int steps = L.degree;
    if (!x0) {
      launch_ew(n, s, [&](int nb, int nt) { jac_first0_kernel<T><<<nb, nt, 0, s>>>(n, dinv, b, w, x); });
      steps -= 1;
    } else {
      to_w(x0);
    }
    for (int it = 0; it < steps; ++it) {
      level_apply(H, L, L.tag, x, y, s);
      launch_ew(n, s, [&](int nb, int nt) { jac_step_kernel<T><<<nb, nt, 0, s>>>(n, dinv, b, y, w, x); });
    }
  }
  if constexpr (sizeof(T) == 8) {
    if (out != (double*)x) launch_ew(n, s, [&](int nb, int nt) { copy_kernel<<<nb, nt, 0, s>>>(n, (const double*)x, out); });
  } else {
    cvt_f32_to_f64(n, (const float*)x, out, s);
  }
}

// Level-0 FP32 smoother on P32 vectors: every step after the first is ONE
// kernel (apply + residual + Chebyshev/Jacobi update, fine_apply_p32_cheb),
// the x iterate ping-pongs between x32 and x32b.  Same FP32 rounding points
// as smooth_t (smoothers.py:90-131).
static void smooth_p32(Hier& H, Level& L, const double* b64, const double* x0, double* out,
                       cudaStream_t s, bool b_ready = false, bool x0_ready = false) {
  const FineOp& op = *H.fine;
  const GridDesc& g = L.g->d;
  const int64_t n = L.n32();
  float* x = L.w.x32.p;
  float* xb = L.w.x32b.p;
  float* d = L.w.dd32.p;
  float* b = L.w.b32.p;
  const float* dinv = L.dinv32p.p;
  static const bool unfused = std::getenv("SG_P32_UNFUSED") != nullptr;  // A/B check
  bool out_done = false;
  // slab window: ghost planes of the iterate before every apply
  auto halo = [&](const float* v) {
    if (H.comm) H.comm->exchange(kP32Level, v, 4, s);
  };
  if (L.kind == 0) {  // Chebyshev
    const double lam = L.lam;
    const double sigma = 0.5 * (lam + L.alpha * lam);
    const double delta = 0.5 * (lam - L.alpha * lam);
    const float c0 = float(1.0 / sigma);
    const int last = L.degree - 1;  // index of the last apply step
    if (!x0) {
      cheb_first0_p32(g, b64, dinv, c0, b, d, x, s);  // b32, d, x in one pass
    } else {
      if (!b_ready) to_p32<double>(g, b64, b, s);
      if (!x0_ready) to_p32<double>(g, x0, x, s);
      halo(x);
      if (unfused) {
        fine_apply_p32(op, x, L.w.y32.p, s);
        launch_ew(n, s, [&](int nb, int nt) { cheb_first_kernel<float><<<nb, nt, 0, s>>>(n, dinv, b, L.w.y32.p, c0, d, x); });
      } else {
        fine_apply_p32_cheb(op, x, xb, b, dinv, d, c0, 0.f, true, s, last == 0 ? out : nullptr);
        out_done = last == 0;
        std::swap(x, xb);
      }
    }
    double a = 2.0 / sigma;
    for (int it = 1; it < L.degree; ++it) {
      const double c = delta * delta * a / 4.0;
      a = 1.0 / (sigma - c);
      halo(x);
      if (unfused) {
        fine_apply_p32(op, x, L.w.y32.p, s);
        const float A = float(a), AC = float(a * c);
        launch_ew(n, s, [&](int nb, int nt) { cheb_step_kernel<float><<<nb, nt, 0, s>>>(n, dinv, b, L.w.y32.p, A, AC, d, x); });
      } else {
        fine_apply_p32_cheb(op, x, xb, b, dinv, d, float(a), float(a * c), false, s,
                            it == last ? out : nullptr);
        out_done = it == last;
        std::swap(x, xb);
      }
    }
  } else {  // damped Jacobi: x = x + w*(dinv*(b - Kx))
    if (!b_ready) to_p32<double>(g, b64, b, s);
    const float w = float(L.omega);
    int steps = L.degree;
    if (!x0) {
      launch_ew(n, s, [&](int nb, int nt) { jac_first0_kernel<float><<<nb, nt, 0, s>>>(n, dinv, b, w, x); });
      steps -= 1;
    } else if (!x0_ready) {
      to_p32<double>(g, x0, x, s);
    }
    for (int it = 0; it < steps; ++it) {
      halo(x);
      fine_apply_p32(op, x, L.w.y32.p, s);
      launch_ew(n, s, [&](int nb, int nt) { jac_step_kernel<float><<<nb, nt, 0, s>>>(n, dinv, b, L.w.y32.p, w, x); });
    }
  }
  L.w.xcur = x;
  if (!out_done && out) from_p32<double>(g, x, out, s);
}

// fused FP64 stencil Chebyshev step / residual on the symmetric copy when
// the level has one (single GPU), else on the full stencil
static void cheb64(Level& L, const double* x, double* xout, const double* b, double* d, double A,
                   double AC, bool first, cudaStream_t s) {
  if (L.st.T64s.p)
    stencil_sym64(*L.g, L.st.T64s.p, 1, x, xout, b, L.dinv.p, d, A, AC, first, s);
  else
    stencil_cheb64(*L.g, L.st.T64.p, x, xout, b, L.dinv.p, d, A, AC, first, s);
}
static void res64(Level& L, const double* x, const double* r, double* out, cudaStream_t s) {
  if (L.st.T64s.p)
    stencil_sym64(*L.g, L.st.T64s.p, 2, x, out, r, nullptr, nullptr, 0.0, 0.0, true, s);
  else
    stencil_res64(*L.g, L.st.T64.p, x, r, out, s);
}

// FP64 Galerkin level, Chebyshev: every apply fused with its update
// (stencil_cheb64); iterates alternate between `out` and the y64 scratch so
// the last lands in `out` and no step reads the buffer it writes.
static bool smooth_st64(Hier& H, Level& L, const double* b, const double* x0, double* out,
                        cudaStream_t s) {
  if (L.is_fine || L.kind != 0 || std::getenv("SG_ST64_UNFUSED")) return false;
  auto halo = [&](const double* v) {  // slab window: ghost planes before every apply
    if (H.comm) H.comm->exchange(L.idx, v, 8, s);
  };
  const int64_t n = L.nd();
  const double lam = L.lam;
  const double sigma = 0.5 * (lam + L.alpha * lam);
  const double delta = 0.5 * (lam - L.alpha * lam);
  const double c0 = 1.0 / sigma;
  const int D = L.degree;
  double* d = L.w.dd64.p;
  double* scratch = L.w.y64.p;
  if (x0 == out || x0 == scratch) return false;
  auto buf = [&](int k) { return ((D - k) & 1) ? scratch : out; };  // iterate X_k
  const double* cur = x0;
  if (!x0) {
    double* x1 = buf(1);
    launch_ew(n, s, [&](int nb, int nt) { cheb_first0_kernel<double><<<nb, nt, 0, s>>>(n, L.dinv.p, b, c0, d, x1); });
    cur = x1;
  } else {
    halo(x0);
    cheb64(L, x0, buf(1), b, d, c0, 0.0, true, s);
    cur = buf(1);
  }
  double a = 2.0 / sigma;
  for (int it = 1; it < D; ++it) {
    const double c = delta * delta * a / 4.0;
    a = 1.0 / (sigma - c);
    halo(cur);
    cheb64(L, cur, buf(it + 1), b, d, a, a * c, false, s);
    cur = buf(it + 1);
  }
  if (D < 1) launch_ew(n, s, [&](int nb, int nt) { copy_kernel<<<nb, nt, 0, s>>>(n, x0, out); });
  return true;
}

void level_smooth(Hier& H, int l, const double* b, const double* x0, double* out, cudaStream_t s) {
  Level& L = *H.lv[size_t(l)];
  if (L.tag == TAG_FP64 && smooth_st64(H, L, b, x0, out, s)) return;
  if (L.p32) {
    smooth_p32(H, L, b, x0, out, s);
    return;
  }
  if (L.tag == TAG_FP64) {
    smooth_t<double>(H, L, b, x0, out, s);
  } else {
    cvt_f64_to_f32(L.nd(), b, L.w.b32.p, s);
    smooth_t<float>(H, L, L.w.b32.p, x0, out, s);
  }
}

void coarsest_solve(Hier& H, const double* r, double* x, cudaStream_t s) {
  if (H.coarsest_mode == 0) H.dense.solve(r, x, s);
  else H.pcg.solve(r, x, s);
}

// hierarchy.py:207-216
static void dist_tail(DistPart& D, int l, int gamma, double* x64, cudaStream_t s);

// On a slab window hierarchy (H.comm / H.dist set) the same recursion runs on
// the windows: every operator input is halo-exchanged first, and below the
// last slab level the replicated coarse tail takes over (dist_tail).
void cycle(Hier& H, int l, int gamma, cudaStream_t s) {
  Level& L = *H.lv[size_t(l)];
  if (l == int(H.lv.size()) - 1 && !H.dist) {
    coarsest_solve(H, L.w.r.p, L.w.x.p, s);
    return;
  }
  Level* Cp = l + 1 < int(H.lv.size()) ? H.lv[size_t(l + 1)].get() : nullptr;
  const int64_t n = L.nd();
  // pre-smoothing writes x (f64) into w.d64 scratch first, then moved to w.x
  double* x64 = L.w.d64.p;  // holds the f64 iterate across the coarse visits
  // V-cycle on a P32 level (one coarse visit, no slab tail below): the f64
  // iterate is never needed as such -- it is f64(x32) exactly before the
  // correction, and the post-smoother starts from f32(x + P e) -- so it is
  // not materialised: the pre-smoother skips its f64 output and the
  // prolongation adds onto f64(x32) in place (SG_P32_X64=1 restores it)
  static const bool keep64 = std::getenv("SG_P32_X64") != nullptr;
  const bool no64 = L.p32 && gamma == 1 && !keep64 && !(H.dist && l + 1 == H.dist->n_dist) &&
                    !std::getenv("SG_P32_UNFUSED");
  if (no64) smooth_p32(H, L, L.w.r.p, nullptr, nullptr, s);
  else level_smooth(H, l, L.w.r.p, nullptr, x64, s);
  for (int g = 0; g < gamma; ++g) {
    if (L.tag == TAG_FP64 && !L.is_fine && !std::getenv("SG_ST64_UNFUSED")) {
      if (H.comm) H.comm->exchange(l, x64, 8, s);
      res64(L, x64, L.w.r.p, L.w.x.p, s);  // r - A x in one pass
    } else if (L.tag == TAG_FP64) {
      level_apply(H, L, TAG_FP64, x64, L.w.y64.p, s);
      launch_ew(n, s, [&](int nb, int nt) { residual_kernel<double><<<nb, nt, 0, s>>>(n, L.w.r.p, L.w.y64.p, L.w.x.p); });
    } else if (L.p32) {
      // x32 = f32(x64): the smoother's last FP32 iterate on the first pass
      // (x64 = f64 of it, so the round trip is exact); re-converted after a
      // coarse correction (W-cycle)
      float* xc = L.w.xcur;
      if (!xc) {  // W-cycle second pass: x32 = f32(x64) was written by prolong
        xc = L.w.x32.p;
      }
      if (H.comm) H.comm->exchange(kP32Level, xc, 4, s);
      fine_apply_p32_res(*H.fine, xc, L.w.r.p, L.w.x.p, s);
    } else {
      cvt_f64_to_f32(n, x64, L.w.x32.p, s);
      level_apply(H, L, L.tag, L.w.x32.p, L.w.y32.p, s);
      launch_ew(n, s, [&](int nb, int nt) { residual_kernel<float><<<nb, nt, 0, s>>>(n, L.w.r.p, L.w.y32.p, L.w.x.p); });
    }
    if (H.comm) H.comm->exchange(l, L.w.x.p, 8, s);  // restriction reads ghost residuals
    if (H.dist && l + 1 == H.dist->n_dist) {
      dist_tail(*H.dist, l, gamma, x64, s);
      if (L.p32) to_p32<double>(L.g->d, x64, L.w.x32.p, s);  // f32(x64) for the post-smoother
    } else {
      Level& C = *Cp;
      restrict_(*L.g, *C.g, L.w.x.p, C.w.r.p, s);  // L.w.x used as residual scratch here
      cycle(H, l + 1, gamma, s);
      if (H.comm) H.comm->exchange(l + 1, C.w.x.p, 8, s);  // prolongation reads ghost corrections
      if (L.p32) {
        // also writes f32(x64) into x32 (P32) for the post-smoother; without
        // the f64 iterate (no64) it adds onto f64(x32) and writes x32 only
        // the iterate may sit in the ping-pong partner: swap the two buffers'
        // roles (a host pointer swap, fixed in the captured graph)
        if (no64 && L.w.xcur != L.w.x32.p) std::swap(L.w.x32, L.w.x32b);
        prolong(*L.g, *C.g, C.w.x.p, no64 ? nullptr : x64, /*add=*/true, s, L.w.x32.p, p32_xs(L.g->d));
      }
      else
        prolong(*L.g, *C.g, C.w.x.p, x64, /*add=*/true, s);
    }
    L.w.xcur = nullptr;  // x64 changed: a W-cycle's next residual re-converts
  }
  if (L.p32) {
    smooth_p32(H, L, L.w.r.p, x64, (l == 0 && H.skip_z64) ? nullptr : L.w.x.p, s,
               /*b_ready=*/true, /*x0_ready=*/true);
    return;
  }
  level_smooth(H, l, L.w.r.p, x64, L.w.x.p, s);
}

Hier::~Hier() {
  for (auto& g : graph)
    if (g) cudaGraphExecDestroy(g);
  if (graph_noz) cudaGraphExecDestroy(graph_noz);
}

const float* cycle_run_noz(Hier& H, cudaStream_t s) {
  SG_REQUIRE(!H.released && H.lv[0]->p32 && !H.dist, "z-in-P32 cycle needs a P32 level 0");
  if (std::getenv("SG_NO_GRAPH")) {
    H.skip_z64 = true;
    try {
      cycle(H, 0, 1, s);
    } catch (...) {
      H.skip_z64 = false;
      throw;
    }
    H.skip_z64 = false;
    return H.lv[0]->w.xcur;
  }
  if (!H.graph_noz) {
    cudaStream_t cs = nullptr;
    SG_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    SG_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    H.skip_z64 = true;
    try {
      cycle(H, 0, 1, cs);
    } catch (...) {
      H.skip_z64 = false;
      cudaStreamEndCapture(cs, &g);
      if (g) cudaGraphDestroy(g);
      cudaStreamDestroy(cs);
      throw;
    }
    H.skip_z64 = false;
    H.zcur32 = H.lv[0]->w.xcur;  // the buffer the captured post-smoother ends in
    SG_CUDA(cudaStreamEndCapture(cs, &g));
    cudaStreamDestroy(cs);
    size_t n = 0;
    SG_CUDA(cudaGraphGetNodes(g, nullptr, &n));
    SG_CUDA(cudaGraphInstantiate(&H.graph_noz, g, 0));
    SG_CUDA(cudaGraphDestroy(g));
    H.graph_noz_nodes = n;
  }
  SG_CUDA(cudaGraphLaunch(H.graph_noz, s));
  __atomic_add_fetch(&g_sg_launches, (unsigned long long)H.graph_noz_nodes, __ATOMIC_RELAXED);
  return H.zcur32;
}

void cycle_run(Hier& H, int gamma, cudaStream_t s) {
  SG_REQUIRE(!H.released, "hierarchy levels were released to a slab solver (single-GPU cycle unavailable)");
  static const bool no_graph = [] {
    const char* e = std::getenv("SG_NO_GRAPH");
    return e && e[0] == '1';
  }();
  SG_REQUIRE(gamma == 1 || gamma == 2, "gamma must be 1 (V) or 2 (W)");
  if (no_graph) {
    cycle(H, 0, gamma, s);
    return;
  }
  if (!H.graph[gamma]) {
    // capture on a private non-blocking stream (the caller's may be the
    // legacy NULL stream, which cannot be captured); capture only records
    cudaStream_t cs = nullptr;
    SG_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    SG_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    try {
      cycle(H, 0, gamma, cs);
    } catch (...) {
      cudaStreamEndCapture(cs, &g);
      if (g) cudaGraphDestroy(g);
      cudaStreamDestroy(cs);
      throw;
    }
    SG_CUDA(cudaStreamEndCapture(cs, &g));
    cudaStreamDestroy(cs);
    size_t n = 0;
    SG_CUDA(cudaGraphGetNodes(g, nullptr, &n));
    SG_CUDA(cudaGraphInstantiate(&H.graph[gamma], g, 0));
    SG_CUDA(cudaGraphDestroy(g));
    H.graph_nodes[gamma] = n;
  }
  SG_CUDA(cudaGraphLaunch(H.graph[gamma], s));
  __atomic_add_fetch(&g_sg_launches, (unsigned long long)H.graph_nodes[gamma], __ATOMIC_RELAXED);
}

// ------------------------------------------------------- diag / power
struct PowerRed {
  const double* dinv;
  double* w;
  const double* v;
  __device__ void operator()(int64_t i, double (&acc)[3]) const {
    const double wv = __dmul_rn(dinv[i], w[i]);
    w[i] = wv;
    acc[0] += v[i] * wv;
    acc[1] += v[i] * v[i];
    acc[2] += wv * wv;
  }
};
struct PowerPost {
  double* sc;  // [0] lam, [1] stop, [2] ww
  __device__ void operator()(const double (&t)[3]) const {
    if (sc[1] != 0.0) return;
    sc[0] = __ddiv_rn(t[0], t[1]);
    sc[2] = t[2];
  }
};
__global__ void power_norm_kernel(int64_t n, const double* __restrict__ w, double* __restrict__ v,
                                  double* __restrict__ sc) {
  SG_ELEMWISE(n);
  if (sc[1] != 0.0) return;
  const double nrm = sqrt(sc[2]);
  if (nrm == 0.0) return;
  v[i_] = __ddiv_rn(w[i_], nrm);
}
__global__ void power_stop_kernel(double* sc) {
  if (sc[1] == 0.0 && sqrt(sc[2]) == 0.0) sc[1] = 1.0;
}

// estimate_lambda_max (smoothers.py:134-152) in FP64 on the level's own operator
static double power_lambda(Hier& H, Level& L, int iters, uint64_t seed, cudaStream_t s) {
  const int64_t n = L.nd();
  double* v = L.w.r.p;
  double* w = L.w.y64.p;
  double* sc = H.scal.p;
  SG_CUDA(cudaMemsetAsync(sc, 0, sizeof(double) * 4, s));
  fill_gaussian_unit(*L.g, seed, v, H.red, sc + 3, s);
  for (int it = 0; it < iters; ++it) {
    level_apply(H, L, TAG_FP64, v, w, s);
    launch_reduce<3>(n, PowerRed{L.dinv.p, w, v}, PowerPost{sc}, H.red, s);
    launch_ew(n, s, [&](int nb, int nt) { power_norm_kernel<<<nb, nt, 0, s>>>(n, w, v, sc); });
    power_stop_kernel<<<1, 1, 0, s>>>(sc);
    SG_CHECK_LAUNCH();
  }
  double lam = 0.0;
  SG_CUDA(cudaMemcpyAsync(&lam, sc, sizeof(double), cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaStreamSynchronize(s));
  return lam > 1e-6 ? lam : 1e-6;
}

void fine_floored_diag(FineOp& op, FineWork& w, cudaStream_t s) {
  if (w.diag_ready) return;
  w.diag.alloc(size_t(3 * op.grid.d.nnodes()));
  fine_diag_raw(op, w.diag.p, s);
  if (!w.scal.p) w.scal.alloc(8);
  np_mean_free(op.grid, w.diag.p, w.scal.p, s);
  diag_floor(op.grid, w.diag.p, w.scal.p, s);
  const int64_t n = 3 * op.grid.d.nnodes();
  w.dinv.alloc(size_t(n));
  DBuf<float> junk(static_cast<size_t>(n));
  launch_ew(n, s, [&](int nb, int nt) { recip_kernel<<<nb, nt, 0, s>>>(n, w.diag.p, w.dinv.p, junk.p); });
  SG_CUDA(cudaStreamSynchronize(s));
  w.diag_ready = true;
}

static void alloc_work(Level& L, cudaStream_t s) {
  const size_t n = size_t(L.nd());
  L.w.r.alloc(n);
  L.w.x.alloc(n);
  L.w.d64.alloc(n);
  L.w.y64.alloc(n);
  L.w.dd64.alloc(n);
  if (L.tag != TAG_FP64) {
    const size_t n32 = L.p32 ? size_t(L.n32()) : n;
    L.w.b32.alloc(n32);
    L.w.x32.alloc(n32);
    L.w.y32.alloc(n32);
    L.w.dd32.alloc(n32);
    if (L.p32) {
      L.w.x32b.alloc(n32);
      // padding entries must read 0 (they are never written)
      for (auto* b : {&L.w.b32, &L.w.x32, &L.w.y32, &L.w.dd32, &L.w.x32b}) b->zero(s);
    }
  }
}

std::unique_ptr<Hier> hier_build(FineOp* fine, FineWork& fw, const HParams& p, const L1Tables& t,
                                 const double* lam_cache, int n_cache, cudaStream_t s) {
  SG_REQUIRE(p.levels >= 1, "need at least one level");
  SG_REQUIRE(p.policy >= 0 && p.policy <= 2, "unknown precision policy");
  auto H = std::make_unique<Hier>();
  H->fine = fine;
  H->policy = p.policy;
  H->emax = fine->emax;
  H->scal.alloc(16);
  H->red.init(s);

  // operators first (hierarchy.py:251-268)
  {
    auto L0 = std::make_unique<Level>();
    L0->idx = 0;
    L0->is_fine = true;
    L0->g = &fine->grid;
    H->lv.push_back(std::move(L0));
  }
  while (int(H->lv.size()) < p.levels) {
    const Grid& cur = *H->lv.back()->g;
    if (cur.d.nx % 2 || cur.d.ny % 2 || cur.d.nz % 2) {
      H->clamped = true;
      break;
    }
    auto C = std::make_unique<Level>();
    C->idx = int(H->lv.size());
    build_coarse_grid(cur, C->own, s);
    if (C->own.n_free == 0) break;
    C->g = &C->own;
    const int64_t nn = C->own.d.nnodes();
    C->st.A64.alloc(size_t(243 * nn));
    if (H->lv.size() == 1) {
      galerkin_level1(*fine, C->own, t, C->st.A64.p, s);
    } else {
      galerkin_next(cur, C->own, H->lv.back()->st.A64.p, C->st.A64.p, s);
    }
    H->lv.push_back(std::move(C));
  }
  const int nl = int(H->lv.size());
  static const int pol[3][3] = {{TAG_FP64, TAG_FP64, TAG_FP64},
                                {TAG_FP32, TAG_FP64, TAG_FP64},
                                {TAG_BF16, TAG_FP32, TAG_FP64}};
  for (int i = 0; i < nl; ++i) {
    Level& L = *H->lv[size_t(i)];
    L.tag = pol[p.policy][std::min(i, 2)];
    L.kind = p.smoother_kind;
    L.degree = i == 0 ? p.degree : p.coarse_smooth_steps;
    L.alpha = p.alpha;
    L.omega = p.omega;
    const size_t n = size_t(L.nd());
    L.diag.alloc(n);
    L.dinv.alloc(n);
    L.dinv32.alloc(n);
    if (L.is_fine) {
      fine_floored_diag(*fine, fw, s);
      launch_ew(int64_t(n), s, [&](int nb, int nt) { copy_kernel<<<nb, nt, 0, s>>>(int64_t(n), fw.diag.p, L.diag.p); });
    } else {
      stencil_diag(*L.g, L.st.A64.p, L.diag.p, s);
      np_mean_free(*L.g, L.diag.p, H->scal.p + 8, s);
      diag_floor(*L.g, L.diag.p, H->scal.p + 8, s);
      if (L.tag == TAG_FP32) {
        L.st.A32.alloc(size_t(243 * L.g->d.nnodes()));
        stencil_round_f32(*L.g, L.st.A64.p, L.st.A32.p, false, s);
        stencil_tile<float>(*L.g, L.st.A32.p, L.st.T32, s);
      }
      stencil_tile<double>(*L.g, L.st.A64.p, L.st.T64, s);
      // single-GPU FP64 smoothing / residual / apply read the symmetric copy
      // (SG_ST64_FULL=1: the full stencil, bit-exact to the reference SpMV)
      if (L.tag == TAG_FP64 && !std::getenv("SG_ST64_FULL")) stencil_sym_tile(*L.g, L.st.A64.p, L.st.T64s, s);
    }
    launch_ew(int64_t(n), s, [&](int nb, int nt) { recip_kernel<<<nb, nt, 0, s>>>(int64_t(n), L.diag.p, L.dinv.p, L.dinv32.p); });
    L.p32 = L.is_fine && L.tag == TAG_FP32 && p32_supported(*fine) && !std::getenv("SG_NO_P32");
    if (L.p32) {  // dinv32 in the P32 layout (0 on padding); the node-layout
                  // copy stays for the slab windows (dist_build)
      L.dinv32p.alloc(size_t(L.n32()));
      L.dinv32p.zero(s);  // the P32 slack past the last plane is never written
      to_p32<float>(L.g->d, L.dinv32.p, L.dinv32p.p, s);
    }
    alloc_work(L, s);
    if (lam_cache && i < n_cache) {
      L.lam = lam_cache[i];
    } else {
      L.lam = 1.1 * power_lambda(*H, L, i == 0 ? 20 : 10, p.power_seed + uint64_t(i), s);
    }
  }

  // coarsest (hierarchy.py:165-178)
  Level& last = *H->lv.back();
  np_mean_free(*last.g, last.diag.p, H->scal.p + 8, s);
  double mean = 0.0;
  SG_CUDA(cudaMemcpyAsync(&mean, H->scal.p + 8, sizeof(double), cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaStreamSynchronize(s));
  H->eps = std::max(mean * 1e-8, 1e-14);
  if (last.is_fine && !last.st.A64.p) {
    last.st.A64.alloc(size_t(243 * last.g->d.nnodes()));
    fine_to_stencil(*fine, last.st.A64.p, s);
  }
  H->coarsest_mode = 1;
  if (last.g->n_free <= p.cholesky_cutoff) {
    SG_REQUIRE(!last.is_fine || last.g->n_free <= 20000,
               "dense assembly limited to 20000 free DOFs");
    DBuf<double> D(size_t(last.g->n_free * last.g->n_free));
    stencil_to_dense(*last.g, last.st.A64.p, D.p, H->eps, s);
    if (H->dense.setup(*last.g, D.p, s)) H->coarsest_mode = 0;
  }
  if (H->coarsest_mode == 1) H->pcg.setup(*last.g, last.st.A64.p, last.diag.p, H->eps, p.coarse_pcg_steps, s);
  const size_t nd0 = size_t(H->lv[0]->nd());
  H->io_a.alloc(nd0);
  H->io_b.alloc(nd0);
  SG_CUDA(cudaStreamSynchronize(s));
  return H;
}

// ------------------------------------------------------ multi-GPU slabs
// Same recursion and rounding points as cycle(); every operator input is
// halo-exchanged first (level_apply through W.comm, explicitly before the
// transfers), so owned rows see exactly the single-GPU operands.  At the
// cut level the residual is allgathered into the replicated full hierarchy,
// the coarse tail runs there, and the prolonged correction (P x_c formed
// first, then added: the bits of prolong(add=true)) is sliced back.
// Below the last slab level: the owned planes of the residual are
// allgathered into the replicated full hierarchy, the coarse tail runs there,
// and the prolonged correction (P x_c formed first, then added: the bits of
// prolong(add=true)) is sliced back into the window iterate x64.
static void dist_tail(DistPart& D, int l, int gamma, double* x64, cudaStream_t s) {
  Hier& F = *D.full;
  Level& L = *D.W->lv[size_t(l)];
  Level& FL = *F.lv[size_t(l)];
  Level& FC = *F.lv[size_t(l + 1)];
  const int64_t n = L.nd();
  D.comm.gather(l, L.w.x.p, FL.w.x.p, s);
  restrict_(*FL.g, *FC.g, FL.w.x.p, FC.w.r.p, s);
  cycle(F, l + 1, gamma, s);
  prolong(*FL.g, *FC.g, FC.w.x.p, FL.w.y64.p, /*add=*/false, s);
  const double* slice = FL.w.y64.p + int64_t(D.w0[l]) * D.plane_nd(l);
  launch_ew(n, s, [&](int nb, int nt) { add_kernel<<<nb, nt, 0, s>>>(n, slice, x64); });
}

void dist_cycle(DistPart& D, int gamma, cudaStream_t s) {
  SG_REQUIRE(gamma == 1 || gamma == 2, "gamma must be 1 (V) or 2 (W)");
  cycle(*D.W, 0, gamma, s);
}

DistPart::~DistPart() {
  for (auto& g : graph)
    if (g) cudaGraphExecDestroy(g);
  if (peer) peer_destroy(peer);
}

// Device transport: no host step inside the cycle, so it is captured once and
// replayed like the single-GPU cycle (cycle_run); host hooks run eagerly.
void dist_cycle_run(DistPart& D, int gamma, cudaStream_t s) {
  static const bool no_graph = [] {
    const char* e = std::getenv("SG_NO_GRAPH");
    return e && e[0] == '1';
  }();
  SG_REQUIRE(gamma == 1 || gamma == 2, "gamma must be 1 (V) or 2 (W)");
  if (no_graph || !D.peer) {
    dist_cycle(D, gamma, s);
    return;
  }
  if (!D.graph[gamma]) {
    cudaStream_t cs = nullptr;
    SG_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    SG_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    try {
      dist_cycle(D, gamma, cs);
    } catch (...) {
      cudaStreamEndCapture(cs, &g);
      if (g) cudaGraphDestroy(g);
      cudaStreamDestroy(cs);
      throw;
    }
    SG_CUDA(cudaStreamEndCapture(cs, &g));
    cudaStreamDestroy(cs);
    size_t n = 0;
    SG_CUDA(cudaGraphGetNodes(g, nullptr, &n));
    SG_CUDA(cudaGraphInstantiate(&D.graph[gamma], g, 0));
    SG_CUDA(cudaGraphDestroy(g));
    D.graph_nodes[gamma] = n;
  }
  SG_CUDA(cudaGraphLaunch(D.graph[gamma], s));
  __atomic_add_fetch(&g_sg_launches, (unsigned long long)D.graph_nodes[gamma], __ATOMIC_RELAXED);
}

void dist_release_full(DistPart& D, cudaStream_t s) {
  SG_CUDA(cudaStreamSynchronize(s));
  Hier& F = *D.full;
  for (int l = 0; l < D.n_dist; ++l) {
    Level& L = *F.lv[size_t(l)];
    const bool cut = l == D.n_dist - 1;
    L.st = Stencil{};
    L.diag.release();
    L.dinv.release();
    L.dinv32.release();
    L.dinv32p.release();
    L.w.r.release();
    L.w.d64.release();
    L.w.dd64.release();
    for (auto* b : {&L.w.b32, &L.w.x32, &L.w.y32, &L.w.dd32, &L.w.x32b}) b->release();
    L.w.xcur = nullptr;
    if (!cut) {
      L.w.x.release();
      L.w.y64.release();
    }
  }
  for (auto& g : F.graph)
    if (g) {
      cudaGraphExecDestroy(g);
      g = nullptr;
    }
  if (F.graph_noz) {
    cudaGraphExecDestroy(F.graph_noz);
    F.graph_noz = nullptr;
  }
  F.io_a.release();
  F.io_b.release();
  D.full_released = true;
  F.released = true;
}

template <class T>
static void copy_planes(const T* src, int64_t src_nn, T* dst, int64_t dst_nn, int64_t node_off,
                        int rows, cudaStream_t s) {
  // dst[q*dst_nn + m] = src[q*src_nn + node_off + m], q < rows (SoA stencil slabs)
  SG_CUDA(cudaMemcpy2DAsync(dst, sizeof(T) * dst_nn, src + node_off, sizeof(T) * src_nn,
                            sizeof(T) * dst_nn, rows, cudaMemcpyDeviceToDevice, s));
}

std::unique_ptr<DistPart> dist_build(Hier& F, int n_dist, const int* planes, const CommHooks& c,
                                     cudaStream_t s) {
  SG_REQUIRE(n_dist >= 1 && n_dist <= 2, "1 or 2 slab-partitioned levels");
  SG_REQUIRE(int(F.lv.size()) > n_dist, "the hierarchy needs a level below the slab levels");
  auto D = std::make_unique<DistPart>();
  D->n_dist = n_dist;
  D->comm = c;
  D->full = &F;
  for (int l = 0; l < n_dist; ++l) {
    D->w0[l] = planes[4 * l + 0];
    D->w1[l] = planes[4 * l + 1];
    D->o0[l] = planes[4 * l + 2];
    D->o1[l] = planes[4 * l + 3];
    SG_REQUIRE(D->w0[l] <= D->o0[l] && D->o0[l] < D->o1[l] && D->o1[l] <= D->w1[l] + 1 &&
                   D->w1[l] <= F.lv[size_t(l)]->g->d.nz,
               "inconsistent slab plan");
  }
  if (n_dist == 2)
    SG_REQUIRE(D->w0[0] == 2 * D->w0[1] && D->w1[0] == std::min(2 * D->w1[1], F.lv[0]->g->d.nz),
               "level-0 window must be the fine image of the level-1 window");
  // level-0 window operator: same element matrix, the window's element layers of E
  const FineOp& ff = *F.fine;
  FineOp& wf = D->wfine;
  build_window_grid(ff.grid, D->w0[0], D->w1[0], wf.grid, s);
  const int64_t layer = int64_t(ff.grid.d.nx) * ff.grid.d.ny;
  const int64_t ne = wf.grid.d.nelem();
  wf.E64.alloc(size_t(ne));
  wf.E32.alloc(size_t(ne));
  SG_CUDA(cudaMemcpyAsync(wf.E64.p, ff.E64.p + D->w0[0] * layer, sizeof(double) * ne, cudaMemcpyDeviceToDevice, s));
  SG_CUDA(cudaMemcpyAsync(wf.E32.p, ff.E32.p + D->w0[0] * layer, sizeof(float) * ne, cudaMemcpyDeviceToDevice, s));
  std::memcpy(wf.ke_host, ff.ke_host, sizeof(wf.ke_host));
  wf.ke64 = ff.ke64;
  wf.ke32 = ff.ke32;
  wf.ke16 = ff.ke16;
  wf.kdiag = ff.kdiag;
  wf.kw64 = ff.kw64;
  wf.kw32 = ff.kw32;
  wf.walsh_ok = ff.walsh_ok;
  wf.emax = ff.emax;
  if (p32_supported(wf)) {  // same FP32 apply arithmetic as the single-GPU level 0
    const size_t n32 = size_t(p32_size(wf.grid.d));
    wf.p32a.alloc(n32);
    wf.p32b.alloc(n32);
    wf.p32a.zero(s);
    wf.p32b.zero(s);
  }

  auto W = std::make_unique<Hier>();
  W->fine = &wf;
  W->policy = F.policy;
  W->emax = F.emax;
  W->comm = &D->comm;
  W->scal.alloc(16);
  W->red.init(s);
  for (int l = 0; l < n_dist; ++l) {
    const Level& FL = *F.lv[size_t(l)];
    auto L = std::make_unique<Level>();
    L->idx = l;
    L->tag = FL.tag;
    L->kind = FL.kind;
    L->degree = FL.degree;
    L->alpha = FL.alpha;
    L->omega = FL.omega;
    L->lam = FL.lam;
    if (l == 0) {
      L->is_fine = true;
      L->g = &wf.grid;
      L->p32 = FL.p32 && p32_supported(wf);  // same FP32 level-0 kernels as one GPU
    } else {
      build_window_grid(*FL.g, D->w0[l], D->w1[l], L->own, s);
      L->g = &L->own;
      const int64_t nnf = FL.g->d.nnodes(), nnw = L->own.d.nnodes();
      const int64_t off = int64_t(D->w0[l]) * (FL.g->d.nx + 1) * (FL.g->d.ny + 1);
      L->st.A64.alloc(size_t(243 * nnw));
      copy_planes(FL.st.A64.p, nnf, L->st.A64.p, nnw, off, 243, s);
      if (FL.st.A32.p) {
        L->st.A32.alloc(size_t(243 * nnw));
        copy_planes(FL.st.A32.p, nnf, L->st.A32.p, nnw, off, 243, s);
        stencil_tile<float>(L->own, L->st.A32.p, L->st.T32, s);
      }
      stencil_tile<double>(L->own, L->st.A64.p, L->st.T64, s);
      // the symmetric copy when the full hierarchy has one: owned rows read
      // their lower blocks from neighbours inside the window (ghost planes)
      if (FL.st.T64s.p) stencil_sym_tile(L->own, L->st.A64.p, L->st.T64s, s);
    }
    const int64_t n = 3 * L->g->d.nnodes();
    const int64_t voff = int64_t(D->w0[l]) * 3 * (FL.g->d.nx + 1) * (FL.g->d.ny + 1);
    L->diag.alloc(size_t(n));
    L->dinv.alloc(size_t(n));
    L->dinv32.alloc(size_t(n));
    SG_CUDA(cudaMemcpyAsync(L->diag.p, FL.diag.p + voff, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    SG_CUDA(cudaMemcpyAsync(L->dinv.p, FL.dinv.p + voff, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    SG_CUDA(cudaMemcpyAsync(L->dinv32.p, FL.dinv32.p + voff, sizeof(float) * n, cudaMemcpyDeviceToDevice, s));
    if (L->p32) {
      L->dinv32p.alloc(size_t(L->n32()));
      L->dinv32p.zero(s);
      to_p32<float>(L->g->d, L->dinv32.p, L->dinv32p.p, s);
    }
    alloc_work(*L, s);
    for (auto* b : {&L->w.r, &L->w.x, &L->w.d64, &L->w.y64, &L->w.dd64}) b->zero(s);
    for (auto* b : {&L->w.b32, &L->w.x32, &L->w.y32, &L->w.dd32, &L->w.x32b}) b->zero(s);
    W->lv.push_back(std::move(L));
  }
  W->dist = D.get();
  D->W = std::move(W);
  // flat-Jacobi scratch of the window operator (1/diag of level 0)
  D->wfw.dinv.alloc(size_t(D->W->lv[0]->nd()));
  SG_CUDA(cudaMemcpyAsync(D->wfw.dinv.p, D->W->lv[0]->dinv.p, sizeof(double) * D->W->lv[0]->nd(),
                          cudaMemcpyDeviceToDevice, s));
  D->wfw.diag_ready = true;
  const size_t ndf = size_t(F.lv[0]->nd());
  D->bfull.alloc(ndf);
  D->xfull.alloc(ndf);
  SG_CUDA(cudaStreamSynchronize(s));
  return D;
}

}  // namespace sg
