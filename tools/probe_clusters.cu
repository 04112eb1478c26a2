// co-resident cluster count for 1-CTA-per-SM kernels (227 KB smem) by cluster size
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k() { extern __shared__ char s[]; if (threadIdx.x == 1024) s[0] = 0; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 6, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 256); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = 220 * 1024;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)k, &cfg);
    printf("cluster %2d: %3d co-resident clusters = %3d SMs (%s)\n", cs, n, n * cs, cudaGetErrorString(e));
  }
  return 0;
}
