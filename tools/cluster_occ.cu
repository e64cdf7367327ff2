// How many clusters of size C (1 CTA/SM, ~225 KB smem) can be co-resident?
#include <cstdio>
__global__ void k(double* p) { extern __shared__ double s[]; s[threadIdx.x] = 1; if (p) p[0] = s[0]; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 230000);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int c : {1, 2, 3, 4, 6, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = c; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1; cfg.blockDim = dim3(256); cfg.gridDim = dim3(c * 16);
    cfg.dynamicSmemBytes = 229376;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster=%2d active=%3d SMs used=%3d (%s)\n", c, n, n * c, cudaGetErrorString(e));
  }
  return 0;
}
