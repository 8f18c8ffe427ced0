// How many clusters of n CTAs (128 threads) can be co-resident on this GPU, for a kernel
// whose dynamic shared memory allows 1, 2 or 3 CTAs per SM (cudaOccupancyMaxActiveClusters).
// Diagnostics for the attention kernel's cluster merge.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) { if (p) p[0] = 1; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("{\"sms\": %d, \"rows\": [\n", sms);
  const int smem[3] = {200 * 1024, 100 * 1024, 70 * 1024};
  bool first = true;
  for (int s = 0; s < 3; ++s)
    for (int n : {1, 2, 4, 8, 12, 16}) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(n, 1, 1);
      cfg.blockDim = dim3(128, 1, 1);
      cfg.dynamicSmemBytes = smem[s];
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = n;
      a[0].val.clusterDim.y = 1;
      a[0].val.clusterDim.z = 1;
      cfg.attrs = a;
      cfg.numAttrs = 1;
      int c = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&c, k, &cfg);
      printf("%s {\"smem_kb\": %d, \"cluster\": %d, \"max_active_clusters\": %d, \"err\": \"%s\"}",
             first ? "" : ",\n", smem[s] / 1024, n, c, cudaGetErrorString(e));
      first = false;
    }
  printf("\n]}\n");
  return 0;
}
