// Development microbenchmark: FP32 pipe rate of scalar FFMA/FADD vs packed
// FFMA2/FADD2 on sm_100a (independent chains, 16 warps per SM).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void __launch_bounds__(512) k(float* out, int iters, float a) {
  float2 x[8];
  for (int i = 0; i < 8; ++i) x[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
  const float2 aa = make_float2(a, a);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) { x[i].x = fmaf(a, x[i].x, 1.0f); x[i].y = fmaf(a, x[i].y, 1.0f); }
      if (MODE == 1) x[i] = __ffma2_rn(aa, x[i], make_float2(1.0f, 1.0f));
      if (MODE == 2) { x[i].x = x[i].x + a; x[i].y = x[i].y + a; }
      if (MODE == 3) x[i] = __fadd2_rn(x[i], aa);
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 4 * 512 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* nm[] = {"FFMA x2", "FFMA2", "FADD x2", "FADD2"};
  for (int m = 0; m < 4; ++m) for (int blocks : {148, 296}) {
    int iters = 20000;
    void (*f)(float*, int, float) = m == 0 ? k<0> : m == 1 ? k<1> : m == 2 ? k<2> : k<3>;
    f<<<blocks, 512>>>(o, 10, 0.999f);
    cudaEventRecord(e0);
    f<<<blocks, 512>>>(o, iters, 0.999f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double lane_ops = double(blocks) * 512 * iters * 16;  // per-lane FP32 ops
    printf("%-8s blocks %d: %.1f T lane-ops/s (%.0f per SM per clk at 1.92 GHz)\n", nm[m], blocks,
           lane_ops / ms / 1e9, lane_ops / (ms * 1e-3) / 148 / 1.92e9);
  }
  return 0;
}
