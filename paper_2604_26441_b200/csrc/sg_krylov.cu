// Native outer solvers: PCG (krylov.py:113-165), restarted FGMRES
// (krylov.py:168-281) and the Lanczos spectral probe (diagnostics.py:38-79).
//
// The host loop here only reads a handful of scalars per iteration (one
// small D2H copy per PCG iteration: pq, rz, ||r||^2 and a step flag); every
// vector operation and reduction runs on the device, deterministically.
#include <chrono>
#include <cmath>
#include <cstdlib>
#include "sg_hier.cuh"
#include "sg_peer.cuh"

namespace sg {

#define SG_EW(n) \
  const int64_t i_ = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; \
  if (i_ >= (n)) return;

namespace {

enum Slot { S_NB = 0, S_PQ, S_RZ, S_RR, S_OK, S_RZN, S_TR, S_BETA, S_TMP, S_H0 = 16 };

struct Dot {
  const double* a;
  const double* b;
  // explicit fma: the fused kernels below must round exactly like this
  __device__ void operator()(int64_t i, double (&acc)[1]) const { acc[0] = fma(a[i], b[i], acc[0]); }
};
struct DiffSq {  // ||b - t||^2
  const double* b;
  const double* t;
  __device__ void operator()(int64_t i, double (&acc)[1]) const {
    const double d = __dsub_rn(b[i], t[i]);
    acc[0] += d * d;
  }
};
struct PcgStep {  // x += a p; r -= a q; rr
  double* x;
  double* r;
  const double* p;
  const double* q;
  const double* sc;
  __device__ void operator()(int64_t i, double (&acc)[1]) const {
    const Ctx c = prep();
    use(i, load(i), c, acc);
  }
  struct V { double x, r, p, q; };
  struct Ctx { double a; bool ok; };
  __device__ Ctx prep() const {  // the step length once per thread, not per element
    const double pq = sc[S_PQ], rz = sc[S_RZ];
    const bool ok = isfinite(pq) && pq != 0.0 && isfinite(rz);
    return {ok ? __ddiv_rn(rz, pq) : 0.0, ok};
  }
  __device__ V load(int64_t i) const { return {x[i], r[i], __ldg(p + i), __ldg(q + i)}; }
  __device__ void use(int64_t i, const V& v, const Ctx& c, double (&acc)[1]) const {
    double rv = v.r;
    if (c.ok) {
      x[i] = __dadd_rn(v.x, __dmul_rn(c.a, v.p));
      rv = __dsub_rn(rv, __dmul_rn(c.a, v.q));
      r[i] = rv;
    }
    acc[0] = fma(rv, rv, acc[0]);
  }
};
struct PcgStepPost {
  double* sc;
  __device__ void operator()(const double (&t)[1]) const {
    const double pq = sc[S_PQ], rz = sc[S_RZ];
    sc[S_OK] = (isfinite(pq) && pq != 0.0 && isfinite(rz)) ? 1.0 : 0.0;
    sc[S_RR] = t[0];
  }
};
struct RznPost {  // beta = rzn/rz ; rz = rzn
  double* sc;
  __device__ void operator()(const double (&t)[1]) const {
    sc[S_RZN] = t[0];
    sc[S_BETA] = __ddiv_rn(t[0], sc[S_RZ]);
    sc[S_RZ] = t[0];
  }
};

__global__ void pupd_kernel(int64_t n, const double* __restrict__ z, double* __restrict__ p,
                            const double* __restrict__ sc) {
  SG_EW(n);
  p[i_] = __dadd_rn(z[i_], __dmul_rn(sc[S_BETA], p[i_]));
}
__global__ void copy_k(int64_t n, const double* __restrict__ a, double* __restrict__ b) {
  SG_EW(n);
  b[i_] = a[i_];
}
__global__ void mul_k(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                      double* __restrict__ c) {
  SG_EW(n);
  c[i_] = __dmul_rn(a[i_], b[i_]);
}
__global__ void sub_k(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                      double* __restrict__ c) {
  SG_EW(n);
  c[i_] = __dsub_rn(a[i_], b[i_]);
}
__global__ void div_host_k(int64_t n, const double* __restrict__ a, double s, double* __restrict__ c) {
  SG_EW(n);
  c[i_] = __ddiv_rn(a[i_], s);
}
__global__ void axpy_dev_k(int64_t n, const double* __restrict__ h, const double* __restrict__ v,
                           double* __restrict__ w) {  // w -= h * v
  SG_EW(n);
  w[i_] = __dsub_rn(w[i_], __dmul_rn(*h, v[i_]));
}
__global__ void gemv_t_k(int64_t n, int J, const double* __restrict__ Q, int64_t ld,
                         const double* __restrict__ h, double* __restrict__ w, double sign) {
  // w = w + sign * (Q^T h) with the GEMV result formed first (numpy: w -= Q.T @ h)
  SG_EW(n);
  double t = 0.0;
  for (int j = 0; j < J; ++j) t += Q[int64_t(j) * ld + i_] * h[j];
  w[i_] = sign > 0 ? __dadd_rn(w[i_], t) : __dsub_rn(w[i_], t);
}
__global__ void f64_to_f32_k(int64_t n, const double* __restrict__ a, float* __restrict__ b) {
  SG_EW(n);
  b[i_] = __double2float_rn(a[i_]);
}
__global__ void f32_to_f64_k(int64_t n, const float* __restrict__ a, double* __restrict__ b) {
  SG_EW(n);
  b[i_] = double(a[i_]);
}

inline int nb256(int64_t n) { return grid_blocks(n, 256); }

// ---------------------------------------------------------------------------
// One GPU: the PCG's reduce-then-update pairs as single cooperative launches.
//  * pq_step: p.q (krylov.py:137), then x += a p, r -= a q and ||r||^2
//    (:138-146) -- p and q are re-read from L2 by the second phase;
//  * rz_pupd: r.z and beta (:158-163), then p = z + beta p (:164).
// Phase 1 and the cross-block sum are exactly reduce_kernel's (same grid,
// same per-thread order, same block tree, partials summed in block order --
// here by every block after a grid barrier instead of by the last block), so
// the results are bit-identical to the separate launches (and to the slab
// path with one rank).  Cooperative launch guarantees co-residency.
// Barrier: thread 0 of each block arrives with a gpu-scope release add and
// polls with acquire loads (the bar.sync on either side orders the block's
// other threads); c_fence_bar = 1 (SG_PCG_FENCE_BAR=1) restores the round-1
// form with two full fences and a __nanosleep back-off.
__constant__ int c_fence_bar;
__device__ __forceinline__ void grid_barrier(unsigned long long* ctr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long nb = gridDim.x;
    if (c_fence_bar) {
      __threadfence();
      const unsigned long long old = atomicAdd(ctr, 1ull);
      const unsigned long long target = (old / nb + 1) * nb;  // counter grows by nb per launch
      while (*(volatile unsigned long long*)ctr < target) __nanosleep(32);
      __threadfence();
    } else {
      unsigned long long old, v;
      asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(ctr) : "memory");
      const unsigned long long target = (old / nb + 1) * nb;
      do {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
      } while (v < target);
    }
  }
  __syncthreads();
}
// last-block election: release of this block's partial, acquire of the others'
__device__ __forceinline__ bool arrive_last(unsigned* counter) {
  if (c_fence_bar) {
    __threadfence();
    return atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(counter) : "memory");
  return old == gridDim.x - 1;
}
// every block: the reduce_kernel last-block sum of partials[0..gridDim)
__device__ __forceinline__ double sum_partials(const double* partials, double* smem, double* bc) {
  double tot[1] = {0.0};
  for (int b = threadIdx.x; b < int(gridDim.x); b += kRedThreads) tot[0] += ((volatile double*)partials)[b];
  __syncthreads();
  block_sum<1>(tot, smem);
  if (threadIdx.x == 0) *bc = tot[0];
  __syncthreads();
  return *bc;
}

__global__ void __launch_bounds__(kRedThreads, 8) pq_step_kernel(int64_t n, double* __restrict__ x,
                                                              double* __restrict__ r,
                                                              const double* __restrict__ p,
                                                              const double* __restrict__ q, double* sc,
                                                              double* partials, unsigned* counter,
                                                              unsigned long long* bar, PeerSumDev ps) {
  __shared__ double smem[8];
  __shared__ double bc;
  __shared__ bool last;
  const int64_t stride = int64_t(gridDim.x) * kRedThreads;
  const int64_t i0 = int64_t(blockIdx.x) * kRedThreads + threadIdx.x;
  double acc[1] = {0.0};
  for (int64_t i = i0; i < n; i += stride) acc[0] = fma(p[i], q[i], acc[0]);  // Dot
  block_sum<1>(acc, smem);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc[0];
  const double rz = sc[S_RZ];
  grid_barrier(bar);
  double pq = sum_partials(partials, smem, &bc);
  if (ps.world > 1) {
    // slab ranks: the rank-ordered sum of the local totals inside this launch
    // (block 0 talks to the peers' mailboxes, the others wait at the barrier)
    if (blockIdx.x == 0 && threadIdx.x == 0) sc[S_PQ] = peer_sum1(ps, pq);
    grid_barrier(bar);
    pq = ((volatile double*)sc)[S_PQ];
  } else if (blockIdx.x == 0 && threadIdx.x == 0) {
    sc[S_PQ] = pq;  // StoreTo
  }
  // PcgStep with this step length (PcgStep::prep / load / use)
  const bool ok = isfinite(pq) && pq != 0.0 && isfinite(rz);
  const double a = ok ? __ddiv_rn(rz, pq) : 0.0;
  // (same accumulation order as PcgStep's four-deep load batches: sequential in i)
  double acc2[1] = {0.0};
  for (int64_t i = i0; i < n; i += stride) {
    double rn = r[i];
    if (ok) {
      x[i] = __dadd_rn(x[i], __dmul_rn(a, p[i]));
      rn = __dsub_rn(rn, __dmul_rn(a, q[i]));
      r[i] = rn;
    }
    acc2[0] = fma(rn, rn, acc2[0]);
  }
  block_sum<1>(acc2, smem);
  double* part2 = partials + gridDim.x;  // phase-1 partials may still be being read
  if (threadIdx.x == 0) {
    part2[blockIdx.x] = acc2[0];
    last = arrive_last(counter);
  }
  __syncthreads();
  if (!last) return;
  if (c_fence_bar) __threadfence();
  double rr = sum_partials(part2, smem, &bc);
  if (threadIdx.x == 0) {  // PcgStepPost, from the values in registers
    if (ps.world > 1) rr = peer_sum1(ps, rr);
    sc[S_OK] = ok ? 1.0 : 0.0;
    sc[S_RR] = rr;
    *counter = 0u;
  }
}

// (slab ranks: the dot runs over the owned range r + off, z + off (n entries),
// the p update over the whole window (nd entries), as the unfused path)
__global__ void __launch_bounds__(kRedThreads, 8) rz_pupd_kernel(int64_t n, int64_t nd, int64_t off,
                                                              const double* __restrict__ r,
                                                              const double* __restrict__ z,
                                                              double* __restrict__ p, double* sc,
                                                              double* partials, unsigned long long* bar,
                                                              PeerSumDev ps) {
  __shared__ double smem[8];
  __shared__ double bc;
  const int64_t stride = int64_t(gridDim.x) * kRedThreads;
  const int64_t i0 = int64_t(blockIdx.x) * kRedThreads + threadIdx.x;
  double acc[1] = {0.0};
  for (int64_t i = i0; i < n; i += stride) acc[0] = fma(r[off + i], z[off + i], acc[0]);  // Dot
  block_sum<1>(acc, smem);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc[0];
  const double rz_old = sc[S_RZ];  // read by every block before block 0 replaces it
  grid_barrier(bar);
  double t = sum_partials(partials, smem, &bc);
  if (ps.world > 1) {  // slab ranks: rank-ordered sum in this launch (see pq_step)
    if (blockIdx.x == 0 && threadIdx.x == 0) sc[S_RZN] = peer_sum1(ps, t);
    grid_barrier(bar);
    t = ((volatile double*)sc)[S_RZN];
  }
  const double beta = __ddiv_rn(t, rz_old);  // RznPost
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    sc[S_RZN] = t;
    sc[S_BETA] = beta;
    sc[S_RZ] = t;
  }
  for (int64_t i = i0; i < nd; i += stride) p[i] = __dadd_rn(z[i], __dmul_rn(beta, p[i]));  // pupd
}

// rz_pupd with z read from the V-cycle's FP32 iterate in the P32 layout
// (sg_fine_pk.cu): z_f64 = f64 of it exactly, so r.z and p = z + beta p carry
// the bits of the node-layout path while the f64 z is never written or read.
struct ZP32 {
  const float* z32;
  int NX, XS;
  __device__ __forceinline__ double operator()(int64_t d) const {
    const int d32 = int(d), node = d32 / 3, c = d32 - 3 * node;
    const int jk = node / NX, i = node - jk * NX;
    return double(z32[(jk * 3 + c) * XS + i]);
  }
};
__global__ void __launch_bounds__(kRedThreads, 8) rz_pupd_z32_kernel(int64_t n, ZP32 Z,
                                                                  const double* __restrict__ r,
                                                                  double* __restrict__ p, double* sc,
                                                                  double* partials,
                                                                  unsigned long long* bar) {
  __shared__ double smem[8];
  __shared__ double bc;
  const int64_t stride = int64_t(gridDim.x) * kRedThreads;
  const int64_t i0 = int64_t(blockIdx.x) * kRedThreads + threadIdx.x;
  double acc[1] = {0.0};
  for (int64_t i = i0; i < n; i += stride) acc[0] = fma(r[i], Z(i), acc[0]);  // Dot
  block_sum<1>(acc, smem);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc[0];
  const double rz_old = sc[S_RZ];
  grid_barrier(bar);
  const double t = sum_partials(partials, smem, &bc);
  const double beta = __ddiv_rn(t, rz_old);  // RznPost
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    sc[S_RZN] = t;
    sc[S_BETA] = beta;
    sc[S_RZ] = t;
  }
  for (int64_t i = i0; i < n; i += stride) p[i] = __dadd_rn(Z(i), __dmul_rn(beta, p[i]));  // pupd
}

struct View {  // non-owning handle on a reused SolverWork buffer
  double* p;
};

template <class Post>
__global__ void post1_kernel(const double* __restrict__ v, Post p) {
  const double t[1] = {*v};
  p(t);
}

struct Ctx {
  NativeSys& sys;
  cudaStream_t s;
  int64_t nd;
  int64_t off = 0, nown = 0;  // reduction range: this rank's owned planes (all of nd on 1 GPU)
  RedWork& red;
  DBuf<double>& sc;
  DBuf<float>& t32a;
  DBuf<float>& t32b;
  Ctx(NativeSys& sy, cudaStream_t st)
      : sys(sy), s(st), red(sy.fw->sw.red), sc(sy.fw->sw.sc), t32a(sy.fw->sw.t32a),
        t32b(sy.fw->sw.t32b) {
    nd = 3 * sys.fine->grid.d.nnodes();
    nown = nd;
    if (sys.dist) {
      off = sys.dist->own_off(0);
      nown = sys.dist->own_n(0);
    }
    red.init(s);
    static const bool fence_bar = [] {  // A/B switch of the grid barrier form (read once)
      if (std::getenv("SG_PCG_FENCE_BAR")) {
        const int one = 1;
        SG_CUDA(cudaMemcpyToSymbol(c_fence_bar, &one, sizeof(int)));
      }
      return true;
    }();
    (void)fence_bar;
    if (!sc.p) sc.alloc(256);
    SG_CUDA(cudaMemsetAsync(sc.p, 0, 256 * sizeof(double), s));
    if (sys.ktag != TAG_FP64 && t32a.n < size_t(nd)) {
      t32a.alloc(size_t(nd));
      t32b.alloc(size_t(nd));
    }
  }
  double* vec(int i) { return sys.fw->sw.vec(i, nd); }
  // y = apply_K(x) promoted to f64 (krylov.py:136: np.asarray(apply_K(p), float64))
  void K(const double* x, double* y) {
    if (sys.dist) sys.dist->comm.exchange(0, x, 8, s);
    if (sys.ktag == TAG_FP64) {
      fine_apply_f64(*sys.fine, x, y, s);
    } else {
      f64_to_f32_k<<<nb256(nd), 256, 0, s>>>(nd, x, t32a.p);
      fine_apply_tag(*sys.fine, sys.ktag, t32a.p, t32b.p, s);
      f32_to_f64_k<<<nb256(nd), 256, 0, s>>>(nd, t32b.p, y);
      SG_CHECK_LAUNCH();
    }
  }
  // fused cooperative reduce-then-update kernels (one GPU); 0 = unavailable
  // slab ranks on the device transport fuse the cross-rank sums into the
  // same launches (PeerSumDev); the host transport cannot
  PeerSumDev psum{};
  bool psum_ok = !sys.dist || peer_sum_dev(sys.dist->peer, psum);
  int fused_blocks() {
    static int per_sm = -1;
    if (!psum_ok || std::getenv("SG_PCG_UNFUSED")) return 0;
    if (per_sm < 0) {
      int a = 0, b = 0, c = 0;
      SG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, pq_step_kernel, kRedThreads, 0));
      SG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, rz_pupd_kernel, kRedThreads, 0));
      SG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, rz_pupd_z32_kernel, kRedThreads, 0));
      per_sm = std::min(a, std::min(b, c));
    }
    const int nb = red_blocks(nown);
    return nb <= per_sm * num_sms() ? nb : 0;
  }
  void pq_step(double* x, double* r, const double* p, const double* q, int nb) {
    // owned range only (slab ranks), as PcgStep in the unfused path
    x += off;
    r += off;
    p += off;
    q += off;
    int64_t n = nown;
    double* scp = sc.p;
    double* part = red.partials.p;
    unsigned* cnt = red.counter.p;
    unsigned long long* bar = red.gbar.p;
    PeerSumDev ps = psum;
    void* args[] = {&n, &x, &r, &p, &q, &scp, &part, &cnt, &bar, &ps};
    SG_CUDA(cudaLaunchCooperativeKernel((const void*)pq_step_kernel, dim3(nb), dim3(kRedThreads), args, 0, s));
    SG_CHECK_LAUNCH();
  }
  void rz_pupd(const double* r, const double* z, double* p, int nb) {
    int64_t n = nown, ndd = nd, o = off;
    double* scp = sc.p;
    double* part = red.partials.p;
    unsigned long long* bar = red.gbar.p;
    PeerSumDev ps = psum;
    void* args[] = {&n, &ndd, &o, &r, &z, &p, &scp, &part, &bar, &ps};
    SG_CUDA(cudaLaunchCooperativeKernel((const void*)rz_pupd_kernel, dim3(nb), dim3(kRedThreads), args, 0, s));
    SG_CHECK_LAUNCH();
  }
  // one GPU, P32 level 0, V-cycle, fused kernels: z stays in FP32 / P32
  bool z32_ok() {
    return sys.hier && !sys.dist && sys.gamma == 1 && sys.hier->lv[0]->p32 && fused_blocks() &&
           !std::getenv("SG_PCG_Z64");
  }
  void M_rz_pupd_z32(const double* r, double* p) {
    Level& L0 = *sys.hier->lv[0];
    if (r != L0.w.r.p) copy_k<<<nb256(nd), 256, 0, s>>>(nd, r, L0.w.r.p);
    ZP32 Z{cycle_run_noz(*sys.hier, s), L0.g->d.nx + 1, p32_xs(L0.g->d)};
    int64_t n = nd;
    double* scp = sc.p;
    double* part = red.partials.p;
    unsigned long long* bar = red.gbar.p;
    void* args[] = {&n, &Z, &r, &p, &scp, &part, &bar};
    SG_CUDA(cudaLaunchCooperativeKernel((const void*)rz_pupd_z32_kernel, dim3(fused_blocks()),
                                        dim3(kRedThreads), args, 0, s));
    SG_CHECK_LAUNCH();
  }
  // z = apply_M(r)
  void M(const double* r, double* z) {
    if (sys.hier) {
      Level& L0 = *sys.hier->lv[0];
      if (r != L0.w.r.p) copy_k<<<nb256(nd), 256, 0, s>>>(nd, r, L0.w.r.p);
      if (sys.dist) dist_cycle_run(*sys.dist, sys.gamma, s);
      else cycle_run(*sys.hier, sys.gamma, s);
      if (z != L0.w.x.p) copy_k<<<nb256(nd), 256, 0, s>>>(nd, L0.w.x.p, z);
    } else {
      mul_k<<<nb256(nd), 256, 0, s>>>(nd, sys.fw->diag_inv_ptr(), r, z);
    }
    SG_CHECK_LAUNCH();
  }
  // reduction of f over the owned range into `slot`, then post(total).  On one
  // GPU this is a single fused launch; on slabs the partial is summed over
  // ranks (rank order) before post runs.
  template <class F, class Post>
  void reduce(const F& f, const Post& post, int slot) {
    if (!sys.dist) {
      launch_reduce<1>(nown, f, post, red, s);
      return;
    }
    launch_reduce<1>(nown, f, StoreTo<1>{{sc.p + slot}}, red, s);
    sys.dist->comm.sum(sc.p + slot, 1, s);
    post1_kernel<<<1, 1, 0, s>>>(sc.p + slot, post);
    SG_CHECK_LAUNCH();
  }
  void dot(const double* a, const double* b, int slot) {
    launch_reduce<1>(nown, Dot{a + off, b + off}, StoreTo<1>{{sc.p + slot}}, red, s);
    if (sys.dist) sys.dist->comm.sum(sc.p + slot, 1, s);
  }
  double read(int slot) {
    double v = 0.0;
    SG_CUDA(cudaMemcpyAsync(&v, sc.p + slot, sizeof(double), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
    return v;
  }
  double true_res(const double* b, const double* x, double* tmp, double normb) {
    K(x, tmp);
    launch_reduce<1>(nown, DiffSq{b + off, tmp + off}, StoreTo<1>{{sc.p + S_TR}}, red, s);
    if (sys.dist) sys.dist->comm.sum(sc.p + S_TR, 1, s);
    return std::sqrt(read(S_TR)) / normb;
  }
};

bool stagnant(const std::vector<double>& best) {  // krylov.py:86-97
  const size_t k = best.size();
  if (k <= 50) return false;
  const double then = best[k - 1 - 50];
  return !(best.back() <= (1.0 - 0.01) * then);
}

void record(std::vector<double>& hist, std::vector<double>& best, double rel) {
  hist.push_back(rel);
  const double prev = best.empty() ? INFINITY : best.back();
  best.push_back(std::min(prev, rel));
}

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

// ------------------------------------------------------------------ PCG
void pcg_native(NativeSys& sys, const double* b, double* x, const SolverCfg& cfg, SolveOut& out,
                std::vector<double>& hist, cudaStream_t s) {
  const double t0 = now();
  Ctx C(sys, s);
  const int64_t nd = C.nd;
  hist.clear();
  std::vector<double> best;
  C.dot(b, b, S_NB);
  const double normb = std::sqrt(C.read(S_NB));
  SG_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * nd, s));
  if (normb == 0.0) {
    out = SolveOut{1, 0, 0.0, 0, now() - t0};
    return;
  }
  // with a hierarchy, r and z ARE the cycle's level-0 input/output vectors
  // (z is consumed by the r.z reduction and the p update before the next
  // cycle overwrites it), so M needs no copies
  const bool alias = sys.hier && !sys.dist;
  const View z{alias ? sys.hier->lv[0]->w.x.p : C.vec(0)}, p{C.vec(1)}, q{C.vec(2)};
  double* r = sys.hier ? sys.hier->lv[0]->w.r.p : C.vec(3);
  copy_k<<<nb256(nd), 256, 0, s>>>(nd, b, r);
  C.M(r, z.p);
  copy_k<<<nb256(nd), 256, 0, s>>>(nd, z.p, p.p);
  SG_CHECK_LAUNCH();
  C.dot(r, z.p, S_RZ);
  double target = cfg.tol;
  int kind = 1;  // cap
  for (int it = 0; it < cfg.maxiter; ++it) {
    C.K(p.p, q.p);
    if (const int fb = C.fused_blocks()) {
      C.pq_step(x, r, p.p, q.p, fb);
    } else {
      C.dot(p.p, q.p, S_PQ);
      C.reduce(PcgStep{x + C.off, r + C.off, p.p + C.off, q.p + C.off, C.sc.p}, PcgStepPost{C.sc.p}, S_TMP);
    }
    double h[4];
    SG_CUDA(cudaMemcpyAsync(h, C.sc.p + S_PQ, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
    const double rz = h[1], rr = h[2], ok = h[3];
    if (!std::isfinite(rz) || ok == 0.0) {  // rz_new / pq checks (krylov.py:138-140, :160-162)
      kind = 3;
      break;
    }
    const double rel = std::sqrt(rr) / normb;
    record(hist, best, rel);
    if (!std::isfinite(rel)) {
      kind = 3;
      break;
    }
    if (rel < target) {
      const double tr = C.true_res(b, x, q.p, normb);
      if (tr < cfg.tol) {
        kind = 0;
        break;
      }
      if (stagnant(best)) {
        kind = 2;
        break;
      }
      target *= 0.1;
    }
    const bool z32 = C.z32_ok();
    if (!z32) C.M(r, z.p);
    if (z32) {
      C.M_rz_pupd_z32(r, p.p);  // z never materialised in f64 (same bits)
    } else if (const int fb = C.fused_blocks()) {
      C.rz_pupd(r, z.p, p.p, fb);
    } else {
      C.reduce(Dot{r + C.off, z.p + C.off}, RznPost{C.sc.p}, S_TMP);
      pupd_kernel<<<nb256(nd), 256, 0, s>>>(nd, z.p, p.p, C.sc.p);
      SG_CHECK_LAUNCH();
    }
    if (it + 1 == cfg.maxiter) {
      // the loop-top check of r.z (krylov.py:160-162) has no next iteration
      // here: a non-finite r.z on the last allowed iteration is non_finite
      double rzn = 0.0;
      SG_CUDA(cudaMemcpyAsync(&rzn, C.sc.p + S_RZ, sizeof(double), cudaMemcpyDeviceToHost, s));
      SG_CUDA(cudaStreamSynchronize(s));
      if (!std::isfinite(rzn)) kind = 3;
    }
  }
  const double tr = C.true_res(b, x, q.p, normb);
  out.converged = std::isfinite(tr) && tr < cfg.tol;
  out.iterations = int(hist.size());
  out.final_true_residual = tr;
  out.failure_kind = out.converged ? 0 : kind;
  out.wall_time = now() - t0;
}

// --------------------------------------------------------------- FGMRES
static void solve_upper(const std::vector<double>& H, int ldh, int n, const std::vector<double>& g,
                        std::vector<double>& y) {
  // back substitution (column-oriented, like reference dtrsv), lstsq fallback
  y.assign(g.begin(), g.begin() + n);
  bool ok = true;
  for (int j = n - 1; j >= 0; --j) {
    const double d = H[size_t(j) * ldh + j];
    y[size_t(j)] = y[size_t(j)] / d;
    const double t = y[size_t(j)];
    for (int i = 0; i < j; ++i) y[size_t(i)] -= t * H[size_t(i) * ldh + j];
  }
  for (double v : y) ok = ok && std::isfinite(v);
  if (ok) return;
  // least squares via Householder QR with column pivoting-free fallback:
  // minimum-norm solution of the (singular) upper system through normal
  // equations regularised at machine precision.
  std::vector<double> A(static_cast<size_t>(n) * n), b(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    b[size_t(i)] = 0.0;
    for (int k = 0; k < n; ++k) {
      double sacc = 0.0;
      for (int r = 0; r < n; ++r) sacc += H[size_t(r) * ldh + i] * H[size_t(r) * ldh + k];
      A[size_t(i) * n + k] = sacc;
    }
    for (int r = 0; r < n; ++r) b[size_t(i)] += H[size_t(r) * ldh + i] * g[size_t(r)];
  }
  double tr = 0.0;
  for (int i = 0; i < n; ++i) tr += A[size_t(i) * n + i];
  for (int i = 0; i < n; ++i) A[size_t(i) * n + i] += 1e-14 * (tr > 0 ? tr : 1.0);
  for (int c = 0; c < n; ++c) {  // Gaussian elimination (SPD)
    const double piv = A[size_t(c) * n + c];
    for (int r = c + 1; r < n; ++r) {
      const double f = A[size_t(r) * n + c] / piv;
      for (int k = c; k < n; ++k) A[size_t(r) * n + k] -= f * A[size_t(c) * n + k];
      b[size_t(r)] -= f * b[size_t(c)];
    }
  }
  for (int r = n - 1; r >= 0; --r) {
    double sacc = b[size_t(r)];
    for (int k = r + 1; k < n; ++k) sacc -= A[size_t(r) * n + k] * y[size_t(k)];
    y[size_t(r)] = sacc / A[size_t(r) * n + r];
  }
}

void fgmres_native(NativeSys& sys, const double* b, double* x, const SolverCfg& cfg, SolveOut& out,
                   std::vector<double>& hist, cudaStream_t s) {
  const double t0 = now();
  Ctx C(sys, s);
  const int64_t nd = C.nd;
  hist.clear();
  std::vector<double> best;
  C.dot(b, b, S_NB);
  const double normb = std::sqrt(C.read(S_NB));
  SG_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * nd, s));
  if (normb == 0.0) {
    out = SolveOut{1, 0, 0.0, 0, now() - t0};
    return;
  }
  const int m = cfg.restart;
  SG_REQUIRE(m + 1 <= 200, "restart too large for the scalar slots");
  SolverWork& sw = sys.fw->sw;
  const View V{SolverWork::grow(sw.basis1, size_t(m + 1) * nd)},
      Z{SolverWork::grow(sw.basis2, size_t(m) * nd)}, w{C.vec(0)}, r{C.vec(1)}, tmp{C.vec(2)},
      yv{SolverWork::grow(sw.small, size_t(m))};
  int kind = 1;
  bool done = false;
  while (!done && int(hist.size()) < cfg.maxiter) {
    C.K(x, tmp.p);
    sub_k<<<nb256(nd), 256, 0, s>>>(nd, b, tmp.p, r.p);
    SG_CHECK_LAUNCH();
    C.dot(r.p, r.p, S_TR);
    const double beta = std::sqrt(C.read(S_TR));
    if (!std::isfinite(beta)) {
      kind = 3;
      break;
    }
    if (beta / normb < cfg.tol) {
      kind = 0;
      break;
    }
    std::vector<double> H(size_t(m + 1) * m, 0.0), cs(size_t(m), 0.0), sn(size_t(m), 0.0),
        g(size_t(m + 1), 0.0);
    g[0] = beta;
    div_host_k<<<nb256(nd), 256, 0, s>>>(nd, r.p, beta, V.p);
    SG_CHECK_LAUNCH();
    int used = 0;
    bool claimed = false;
    for (int j = 0; j < m; ++j) {
      double* Vj = V.p + int64_t(j) * nd;
      double* Zj = Z.p + int64_t(j) * nd;
      C.M(Vj, Zj);
      C.K(Zj, w.p);
      for (int i = 0; i <= j; ++i) {  // modified Gram-Schmidt
        const double* Vi = V.p + int64_t(i) * nd;
        C.dot(w.p, Vi, S_H0 + i);
        axpy_dev_k<<<nb256(nd), 256, 0, s>>>(nd, C.sc.p + S_H0 + i, Vi, w.p);
        SG_CHECK_LAUNCH();
      }
      C.dot(w.p, w.p, S_H0 + j + 1);
      std::vector<double> col(size_t(j + 2));
      SG_CUDA(cudaMemcpyAsync(col.data(), C.sc.p + S_H0, sizeof(double) * (j + 2),
                              cudaMemcpyDeviceToHost, s));
      SG_CUDA(cudaStreamSynchronize(s));
      col[size_t(j + 1)] = std::sqrt(col[size_t(j + 1)]);
      bool fin = true;
      for (int i = 0; i <= j + 1; ++i) {
        H[size_t(i) * m + j] = col[size_t(i)];
        fin = fin && std::isfinite(col[size_t(i)]);
      }
      if (!fin) {
        kind = 3;
        done = true;
        used = j + 1;
        break;
      }
      const bool happy = H[size_t(j + 1) * m + j] < 1e-14;
      if (!happy) {
        div_host_k<<<nb256(nd), 256, 0, s>>>(nd, w.p, H[size_t(j + 1) * m + j], V.p + int64_t(j + 1) * nd);
        SG_CHECK_LAUNCH();
      }
      for (int i = 0; i < j; ++i) {
        const double h0 = cs[size_t(i)] * H[size_t(i) * m + j] + sn[size_t(i)] * H[size_t(i + 1) * m + j];
        H[size_t(i + 1) * m + j] = -sn[size_t(i)] * H[size_t(i) * m + j] + cs[size_t(i)] * H[size_t(i + 1) * m + j];
        H[size_t(i) * m + j] = h0;
      }
      const double den = std::hypot(H[size_t(j) * m + j], H[size_t(j + 1) * m + j]);
      if (den == 0.0) {
        cs[size_t(j)] = 1.0;
        sn[size_t(j)] = 0.0;
      } else {
        cs[size_t(j)] = H[size_t(j) * m + j] / den;
        sn[size_t(j)] = H[size_t(j + 1) * m + j] / den;
      }
      H[size_t(j) * m + j] = cs[size_t(j)] * H[size_t(j) * m + j] + sn[size_t(j)] * H[size_t(j + 1) * m + j];
      H[size_t(j + 1) * m + j] = 0.0;
      g[size_t(j + 1)] = -sn[size_t(j)] * g[size_t(j)];
      g[size_t(j)] = cs[size_t(j)] * g[size_t(j)];
      used = j + 1;
      const double rel = std::fabs(g[size_t(j + 1)]) / normb;
      record(hist, best, rel);
      if (!std::isfinite(rel)) {
        kind = 3;
        done = true;
        break;
      }
      if (happy || rel < cfg.tol) {
        claimed = true;
        break;
      }
      if (int(hist.size()) >= cfg.maxiter) break;
    }
    if (kind == 3) break;
    if (used > 0) {
      std::vector<double> Hs(size_t(used) * used), y;
      for (int i = 0; i < used; ++i)
        for (int k = 0; k < used; ++k) Hs[size_t(i) * used + k] = H[size_t(i) * m + k];
      solve_upper(Hs, used, used, g, y);
      SG_CUDA(cudaMemcpyAsync(yv.p, y.data(), sizeof(double) * used, cudaMemcpyHostToDevice, s));
      gemv_t_k<<<nb256(nd), 256, 0, s>>>(nd, used, Z.p, nd, yv.p, x, 1.0);
      SG_CHECK_LAUNCH();
    }
    if (done) break;
    const double tr = C.true_res(b, x, tmp.p, normb);
    if (tr < cfg.tol) {
      kind = 0;
      break;
    }
    if (claimed && stagnant(best)) {
      kind = 2;
      break;
    }
    if (int(hist.size()) >= cfg.maxiter) {
      kind = 1;
      break;
    }
  }
  const double tr = C.true_res(b, x, tmp.p, normb);
  out.converged = std::isfinite(tr) && tr < cfg.tol;
  out.iterations = int(hist.size());
  out.final_true_residual = tr;
  out.failure_kind = out.converged ? 0 : kind;
  out.wall_time = now() - t0;
}

// One slab-partitioned operator application on this rank's window vectors
// (what 0: y = K_ktag x, what 1: y = M x).
void dist_apply(NativeSys& sys, int what, const double* xw, double* yw, cudaStream_t s) {
  SG_REQUIRE(sys.dist, "not a slab system");
  Ctx C(sys, s);
  if (what == 0) C.K(xw, yw);
  else C.M(xw, yw);
}

// -------------------------------------------------------------- Lanczos
void lanczos_native(NativeSys& sys, int m, uint64_t seed, std::vector<double>& H, int& used,
                    bool& partial, cudaStream_t s) {
  SG_REQUIRE(!sys.dist, "the Lanczos probe is single-GPU");
  Ctx C(sys, s);
  const int64_t nd = C.nd;
  SG_REQUIRE(m >= 2 && m <= 200, "Lanczos steps out of range");
  const View Q{SolverWork::grow(sys.fw->sw.basis1, size_t(m) * nd)}, w{C.vec(0)}, kv{C.vec(1)};
  H.assign(size_t(m) * m, 0.0);
  used = m;
  partial = false;
  fill_gaussian_unit(sys.fine->grid, seed, Q.p, C.red, C.sc.p + S_TR, s);
  for (int j = 0; j < m; ++j) {
    const double* Qj = Q.p + int64_t(j) * nd;
    C.K(Qj, kv.p);
    C.M(kv.p, w.p);
    for (int t = 0; t <= j; ++t) C.dot(Q.p + int64_t(t) * nd, w.p, S_H0 + t);
    gemv_t_k<<<nb256(nd), 256, 0, s>>>(nd, j + 1, Q.p, nd, C.sc.p + S_H0, w.p, -1.0);
    SG_CHECK_LAUNCH();
    std::vector<double> h(size_t(j + 1)), h2(size_t(j + 1));
    SG_CUDA(cudaMemcpyAsync(h.data(), C.sc.p + S_H0, sizeof(double) * (j + 1), cudaMemcpyDeviceToHost, s));
    for (int t = 0; t <= j; ++t) C.dot(Q.p + int64_t(t) * nd, w.p, S_H0 + t);
    gemv_t_k<<<nb256(nd), 256, 0, s>>>(nd, j + 1, Q.p, nd, C.sc.p + S_H0, w.p, -1.0);
    SG_CHECK_LAUNCH();
    SG_CUDA(cudaMemcpyAsync(h2.data(), C.sc.p + S_H0, sizeof(double) * (j + 1), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
    for (int t = 0; t <= j; ++t) H[size_t(t) * m + j] = h[size_t(t)] + h2[size_t(t)];
    if (j == m - 1) break;
    C.dot(w.p, w.p, S_TR);
    const double bn = std::sqrt(C.read(S_TR));
    if (!std::isfinite(bn) || bn < 1e-14) {
      used = j + 1;
      partial = true;
      break;
    }
    H[size_t(j + 1) * m + j] = bn;
    div_host_k<<<nb256(nd), 256, 0, s>>>(nd, w.p, bn, Q.p + int64_t(j + 1) * nd);
    SG_CHECK_LAUNCH();
  }
}

}  // namespace sg
