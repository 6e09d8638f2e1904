// Development microbenchmark: cost of one deterministic grid all-reduce of a
// double across one block per SM (the pcg80 inner barrier), for several
// publish/poll schemes.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

struct Args { unsigned* bar; double* part; uint4* slots; int stride; int reps; double* out; };

__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int V>
__global__ void __launch_bounds__(432, 1) k(Args A) {
  __shared__ double red[32];
  __shared__ double tot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int nb = gridDim.x;
  double acc = 0.0;
  double v = 1.0 + threadIdx.x * 1e-3 + blockIdx.x;
  for (int e = 1; e <= A.reps; ++e) {
    double w = wsum(v);
    if (lane == 0) red[warp] = w;
    __syncthreads();
    if (V >= 8) {  // counter barrier, relaxed polling; V9: + fences; V10: + warp-tree local sums
      double* part = A.part + (e & 1) * nb;
      if (warp == 0) {
        double s;
        if (V >= 10) { s = lane < nw ? red[lane] : 0.0; s = wsum(s); }
        else { s = 0; if (lane == 0) for (int i = 0; i < nw; ++i) s += red[i]; }
        if (lane == 0) {
          __stcg(part + blockIdx.x, s);
          if (V == 9 || V == 10) __threadfence();
          if (V == 12) asm volatile("fence.acq_rel.gpu;" ::: "memory");
          if (V == 11) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(A.bar) : "memory");
          else asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(A.bar) : "memory");
          unsigned f, target = unsigned(e) * nb;
          do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(A.bar) : "memory"); } while (f < target);
        }
        __syncwarp();
        if (V >= 9) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        double a[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) { const int b = lane + 32 * q; a[q] = b < nb ? __ldcg(part + b) : 0.0; }
        double t = a[0] + a[1] + a[2] + a[3] + a[4];
        t = wsum(t);
        if (lane == 0) tot = t;
      }
    } else if (V == 6) {  // block-local only (loop floor)
      if (threadIdx.x == 0) { double s = 0; for (int i = 0; i < nw; ++i) s += red[i]; tot = s; }
    } else if (V == 7) {  // counter only, one poller, no partials
      if (threadIdx.x == 0) {
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(A.bar) : "memory");
        unsigned f, target = unsigned(e) * nb;
        do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(A.bar) : "memory"); } while (f < target);
        tot = red[0];
      }
    } else if (V == 0) {  // counter barrier + partial reads
      double* part = A.part + (e & 1) * nb;
      if (threadIdx.x == 0) {
        double s = 0; for (int i = 0; i < nw; ++i) s += red[i];
        __stcg(part + blockIdx.x, s);
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(A.bar) : "memory");
        unsigned f, target = unsigned(e) * nb;
        do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(A.bar) : "memory"); } while (f < target);
      }
      __syncthreads();
      if (warp == 0) {
        double t = 0;
        for (int b = lane; b < nb; b += 32) t += __ldcg(part + b);
        t = wsum(t);
        if (lane == 0) tot = t;
      }
    } else if (V >= 4) {  // master gather + broadcast (V4: per-block inbox, V5: one line)
      const unsigned flag = unsigned(e);
      uint4* sl = A.slots + size_t(e & 1) * nb * A.stride;        // arrivals
      uint4* ib = A.slots + size_t(2 + (e & 1)) * nb * A.stride;  // inboxes / broadcast
      if (warp == 0) {
        if (lane == 0) {
          double s = 0; for (int i = 0; i < nw; ++i) s += red[i];
          unsigned lo = __double2loint(s), hi = __double2hiint(s);
          asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(sl + size_t(blockIdx.x) * A.stride),
                       "r"(lo), "r"(flag), "r"(hi), "r"(flag) : "memory");
        }
        if (blockIdx.x == 0) {
          double a[5];
          bool done;
          do {
            done = true;
#pragma unroll
            for (int q = 0; q < 5; ++q) {
              const int b = lane + 32 * q;
              a[q] = 0.0;
              if (b < nb) {
                unsigned x0, f0, x1, f1;
                asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x0), "=r"(f0), "=r"(x1), "=r"(f1) : "l"(sl + size_t(b) * A.stride) : "memory");
                done = done && f0 == flag && f1 == flag;
                a[q] = __hiloint2double(int(x1), int(x0));
              }
            }
          } while (!__all_sync(0xffffffffu, done));
          double t = a[0] + a[1] + a[2] + a[3] + a[4];
          t = wsum(t);
          unsigned lo = __double2loint(t), hi = __double2hiint(t);
          if (V == 4) {
            for (int b = lane; b < nb; b += 32)
              asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(ib + size_t(b) * A.stride),
                           "r"(lo), "r"(flag), "r"(hi), "r"(flag) : "memory");
          } else if (lane == 0) {
            asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(ib),
                         "r"(lo), "r"(flag), "r"(hi), "r"(flag) : "memory");
          }
        }
        if (lane == 0) {
          const uint4* src = V == 4 ? ib + size_t(blockIdx.x) * A.stride : ib;
          unsigned x0, f0, x1, f1;
          do {
            asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x0), "=r"(f0), "=r"(x1), "=r"(f1) : "l"(src) : "memory");
          } while (f0 != flag || f1 != flag);
          tot = __hiloint2double(int(x1), int(x0));
        }
      }
    } else {  // LL packets
      const unsigned flag = unsigned(e);
      uint4* sl = A.slots + size_t(e & 1) * nb * A.stride;
      if (warp == 0) {
        if (lane == 0) {
          double s = 0; for (int i = 0; i < nw; ++i) s += red[i];
          if (V == 2) __threadfence();
          unsigned lo = __double2loint(s), hi = __double2hiint(s);
          asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(sl + size_t(blockIdx.x) * A.stride),
                       "r"(lo), "r"(flag), "r"(hi), "r"(flag) : "memory");
        }
        double a[5];
        bool done;
        do {
          done = true;
#pragma unroll
          for (int q = 0; q < 5; ++q) {
            const int b = lane + 32 * q;
            a[q] = 0.0;
            if (b < nb) {
              unsigned x0, f0, x1, f1;
              if (V == 3)
                asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x0), "=r"(f0), "=r"(x1), "=r"(f1) : "l"(sl + size_t(b) * A.stride) : "memory");
              else
                asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x0), "=r"(f0), "=r"(x1), "=r"(f1) : "l"(sl + size_t(b) * A.stride) : "memory");
              done = done && f0 == flag && f1 == flag;
              a[q] = __hiloint2double(int(x1), int(x0));
            }
          }
        } while (!__all_sync(0xffffffffu, done));
        if (V == 2) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        double t = a[0] + a[1] + a[2] + a[3] + a[4];
        t = wsum(t);
        if (lane == 0) tot = t;
      }
    }
    __syncthreads();
    acc += tot;
    v = acc * 1e-30 + v;
  }
  if (threadIdx.x == 0) A.out[blockIdx.x] = acc;
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int nb = 147;
  Args a; a.reps = 2000;
  cudaMalloc(&a.bar, 64); cudaMalloc(&a.part, 2 * 256 * 8); cudaMalloc(&a.out, 256 * 8);
  cudaMalloc(&a.slots, 4 * 256 * 8 * sizeof(uint4));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"counter+partials", "LL packed/volatile", "LL +fences", "LL relaxed.gpu",
                         "master+inboxes", "master+1 line", "block-local floor", "counter relaxed only", "counter+partials relaxed", "  + fences", "  + warp-tree local", "red.release+acq_rel", "acq_rel x2"};
  for (int V = 0; V < 13; ++V)
    for (int stride : {1, 8}) {
      if ((V == 0 || V >= 6) && stride == 8) continue;
      if (V >= 1 && V <= 5) continue;
      a.stride = stride;
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(a.bar, 0, 64); cudaMemset(a.slots, 0, 4 * 256 * 8 * sizeof(uint4));
        void* args[] = {&a};
        void* fn = V == 0 ? (void*)k<0> : V == 1 ? (void*)k<1> : V == 2 ? (void*)k<2> : V == 3 ? (void*)k<3> : V == 4 ? (void*)k<4> : V == 5 ? (void*)k<5> : V == 6 ? (void*)k<6> : V == 7 ? (void*)k<7> : V == 8 ? (void*)k<8> : V == 9 ? (void*)k<9> : V == 10 ? (void*)k<10> : V == 11 ? (void*)k<11> : (void*)k<12>;
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel(fn, dim3(nb), dim3(432), args, 0, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep) printf("%-22s stride %d: %.3f us per all-reduce (%s)\n", names[V], stride, ms * 1e3 / a.reps,
                        cudaGetErrorString(cudaGetLastError()));
      }
    }
  return 0;
}
