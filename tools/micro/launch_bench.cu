// Launch / dispatch cost of a pcg80-shaped kernel (147 blocks x 448 threads,
// ~200 KB dynamic shared memory, optional 512-column TMEM allocation), normal
// vs cooperative launch, and after a small default-carveout kernel.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_bench launch_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int TMEM>
__global__ void __launch_bounds__(448, 1) big_k(int* out) {
  extern __shared__ double sm[];
  __shared__ unsigned tm;
  if (TMEM) {
    if (threadIdx.x < 32) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       static_cast<unsigned>(__cvta_generic_to_shared(&tm))) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0 && sm[5] < 0) out[blockIdx.x] = 1;
  if (TMEM) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
  }
}
__global__ void small_k(int* out) {
  if (threadIdx.x == 0 && blockIdx.x > 100000) out[0] = 1;
}

int main() {
  int* d;
  cudaMalloc(&d, 4096);
  const int smem = 200 * 1024, nb = 147, n = 200;
  cudaFuncSetAttribute(big_k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(big_k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(a, s);
    for (int i = 0; i < n; ++i) launch();
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-48s %8.2f us per iteration\n", name, 1e3f * ms / n);
  };
  void* args[] = {&d};
  run("small kernel (148 x 128)", [&] { small_k<<<148, 128, 0, s>>>(d); });
  run("big normal", [&] { big_k<0><<<nb, 448, smem, s>>>(d); });
  run("big cooperative", [&] {
    cudaLaunchCooperativeKernel((void*)big_k<0>, dim3(nb), dim3(448), args, smem, s);
  });
  run("big cooperative + TMEM", [&] {
    cudaLaunchCooperativeKernel((void*)big_k<1>, dim3(nb), dim3(448), args, smem, s);
  });
  run("big normal + TMEM", [&] { big_k<1><<<nb, 448, smem, s>>>(d); });
  run("small + big normal", [&] {
    small_k<<<148, 128, 0, s>>>(d);
    big_k<0><<<nb, 448, smem, s>>>(d);
  });
  run("small + big cooperative + TMEM", [&] {
    small_k<<<148, 128, 0, s>>>(d);
    cudaLaunchCooperativeKernel((void*)big_k<1>, dim3(nb), dim3(448), args, smem, s);
  });
  // the same pairs captured in a graph (as in the V-cycle)
  auto graph_run = [&](const char* name, auto body) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < 20; ++i) body();
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(a, s);
    for (int i = 0; i < 10; ++i) cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-48s %8.2f us per iteration\n", name, 1e3f * ms / 200);
  };
  graph_run("graph: small", [&] { small_k<<<148, 128, 0, s>>>(d); });
  graph_run("graph: small + small", [&] { small_k<<<148, 128, 0, s>>>(d); small_k<<<148, 128, 0, s>>>(d); });
  graph_run("graph: small + big normal + TMEM", [&] {
    small_k<<<148, 128, 0, s>>>(d);
    big_k<1><<<nb, 448, smem, s>>>(d);
  });
  graph_run("graph: small + big cooperative + TMEM", [&] {
    small_k<<<148, 128, 0, s>>>(d);
    cudaLaunchCooperativeKernel((void*)big_k<1>, dim3(nb), dim3(448), args, smem, s);
  });
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
