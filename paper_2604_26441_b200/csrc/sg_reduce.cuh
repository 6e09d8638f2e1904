// Deterministic multi-value reductions (PCG dots / norms, smoother norms).
//
// One launch: every block reduces a fixed grid-stride slice with a fixed
// shuffle tree, writes its partial, and the last block to arrive sums the
// partials in index order.  The result bits depend only on n and the grid
// size (fixed per n), never on block scheduling -- the reference's
// determinism contract (test_acceptance.py:244-257).
#pragma once
#include <type_traits>
#include "sg_common.cuh"

namespace sg {

constexpr int kRedThreads = 256;
constexpr int kRedMaxBlocks = 1184;  // 8 blocks per SM

inline int red_blocks(int64_t n) {
  int64_t b = (n + kRedThreads * 4 - 1) / (kRedThreads * 4);
  if (b < 1) b = 1;
  if (b > kRedMaxBlocks) b = kRedMaxBlocks;
  return int(b);
}

struct RedWork {
  DBuf<double> partials;  // kRedMaxBlocks * 8
  DBuf<unsigned> counter;
  DBuf<unsigned long long> gbar;  // grid barrier of the fused PCG kernels (monotonic)
  void init(cudaStream_t s) {
    if (!partials.p) {
      partials.alloc(size_t(kRedMaxBlocks) * 8);
      counter.alloc(1);
      counter.zero(s);
      gbar.alloc(1);
      gbar.zero(s);
    }
  }
};

template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* smem /* NV*8 */) {
#pragma unroll
  for (int k = 0; k < NV; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) smem[k * 8 + warp] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = smem[k * 8 + 0];
      for (int w = 1; w < kRedThreads / 32; ++w) s += smem[k * 8 + w];
      v[k] = s;
    }
  }
}

// F: __device__ void operator()(int64_t i, double (&acc)[NV]) const  (adds into acc)
// Post: __device__ void operator()(const double (&tot)[NV]) const    (run once, thread 0 of last block)
//
// Split functors (the hot PCG ones) also define V (an element's loaded
// operands), Ctx (per-thread constants, e.g. a step length computed once
// instead of per element), prep(), load(i) and use(i, v, ctx, acc): the
// kernel then issues four elements' loads before accumulating them -- in the
// same order as the plain loop, so the result bits are unchanged.
template <class F, class = void>
struct SplitRed : std::false_type {};
template <class F>
struct SplitRed<F, std::void_t<typename F::V>> : std::true_type {};

template <int NV, class F>
__device__ __forceinline__ void red_loop(const F& f, int64_t n, double (&acc)[NV]) {
  const int64_t stride = int64_t(gridDim.x) * kRedThreads;
  int64_t i = int64_t(blockIdx.x) * kRedThreads + threadIdx.x;
  if constexpr (SplitRed<F>::value) {
    const typename F::Ctx ctx = f.prep();
    for (; i + 3 * stride < n; i += 4 * stride) {
      const typename F::V v0 = f.load(i), v1 = f.load(i + stride), v2 = f.load(i + 2 * stride),
                          v3 = f.load(i + 3 * stride);
      f.use(i, v0, ctx, acc);
      f.use(i + stride, v1, ctx, acc);
      f.use(i + 2 * stride, v2, ctx, acc);
      f.use(i + 3 * stride, v3, ctx, acc);
    }
    for (; i < n; i += stride) f.use(i, f.load(i), ctx, acc);
  } else {
    for (; i < n; i += stride) f(i, acc);
  }
}

template <int NV, class F, class Post>
__global__ void __launch_bounds__(kRedThreads) reduce_kernel(int64_t n, F f, Post post,
                                                             double* partials, unsigned* counter) {
  __shared__ double smem[NV * 8];
  __shared__ bool last;
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;
  red_loop<NV>(f, n, acc);
  block_sum<NV>(acc, smem);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) partials[blockIdx.x * NV + k] = acc[k];
    __threadfence();
    unsigned t = atomicAdd(counter, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double tot[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) tot[k] = 0.0;
  for (int b = threadIdx.x; b < int(gridDim.x); b += kRedThreads) {
#pragma unroll
    for (int k = 0; k < NV; ++k) tot[k] += ((volatile double*)partials)[b * NV + k];
  }
  __syncthreads();
  block_sum<NV>(tot, smem);
  if (threadIdx.x == 0) {
    post(tot);
    *counter = 0u;
  }
}

template <int NV, class F, class Post>
inline void launch_reduce(int64_t n, const F& f, const Post& post, RedWork& w, cudaStream_t s) {
  w.init(s);
  int nb = red_blocks(n);
  reduce_kernel<NV, F, Post><<<nb, kRedThreads, 0, s>>>(n, f, post, w.partials.p, w.counter.p);
  SG_CHECK_LAUNCH();
}

// Post functor: store the totals to device scalars.
template <int NV>
struct StoreTo {
  double* dst[NV];
  __device__ void operator()(const double (&t)[NV]) const {
#pragma unroll
    for (int k = 0; k < NV; ++k)
      if (dst[k]) *dst[k] = t[k];
  }
};

}  // namespace sg
