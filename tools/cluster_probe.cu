// How many clusters of a given size fit at once on this GPU when every CTA
// needs a whole SM (198 KB of shared memory), vs the SM count: the cost of
// giving a lane group cluster residency instead of a cooperative launch.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void big_smem_kernel(int* out) {
  extern __shared__ int s[];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0 && s[1] == 12345) out[0] = 1;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int smem = 198 * 1024;
  cudaFuncSetAttribute(big_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(big_smem_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  printf("SMs %d\n", p.multiProcessorCount);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = cs;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, big_smem_kernel, &cfg);
    printf("cluster %2d: max active clusters %d (%d SMs used) %s\n", cs, n, n * cs,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
