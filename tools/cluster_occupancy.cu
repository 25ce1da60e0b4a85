// Max active clusters vs cluster size for a 512-thread CTA with ~218 KB of dynamic shared memory
// (the tensor-core filter's footprint): how many SMs each cluster size can keep busy on this GPU.
#include <cstdio>
__global__ void k(int* p) { extern __shared__ int s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }
int main() {
  const int smem = 223232;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d\n", sms);
  for (int c = 1; c <= 16; ++c) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = c; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(512); cfg.gridDim = dim3(c); cfg.dynamicSmemBytes = smem; cfg.attrs = a; cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %2d: max active clusters %3d -> %3d SMs (%s)\n", c, n, n * c, cudaGetErrorString(e));
  }
  return 0;
}
