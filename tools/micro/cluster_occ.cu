// Thread-block cluster residency for a one-CTA-per-SM kernel shaped like the
// pcg80 brick kernel (448 threads, > 114 KB of shared memory, so exactly one
// CTA fits an SM): cudaOccupancyMaxActiveClusters for cluster sizes 1..16.
// The brick kernel needs all of its 147 CTAs co-resident (grid-wide
// all-reduce every step), so a clustered launch is possible only for a size
// whose max-active-clusters x size >= the brick count.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o cluster_occ cluster_occ.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(448, 1) brick_like(int* out) {
  extern __shared__ int sm[];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0 && out) out[blockIdx.x] = sm[1];
}

int main() {
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int smem = 160 * 1024;
  cudaFuncSetAttribute(brick_like, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(brick_like, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  printf("SMs %d, 448 threads, %d KB dynamic shared memory per CTA\n", nsm, smem / 1024);
  for (int cs = 1; cs <= 16; ++cs) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64, 1, 1);
    cfg.blockDim = dim3(448, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    const cudaError_t e = cudaOccupancyMaxActiveClusters(&n, brick_like, &cfg);
    if (e != cudaSuccess) {
      printf("cluster %2d: %s\n", cs, cudaGetErrorString(e));
      cudaGetLastError();
      continue;
    }
    printf("cluster %2d: max active clusters %3d -> %3d co-resident CTAs\n", cs, n, n * cs);
  }
  return 0;
}
