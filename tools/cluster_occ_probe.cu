// Max co-resident thread-block clusters on this GPU per cluster size and shared-memory footprint
// (cudaOccupancyMaxActiveClusters): which cluster shapes can occupy all SMs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/cluster_occ_probe tools/cluster_occ_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k256(float* o) { extern __shared__ float s[]; if (o) o[0] = s[0]; }
__global__ void __launch_bounds__(512, 1) k512(float* o) { extern __shared__ float s[]; if (o) o[0] = s[0]; }
template <typename F>
static void probe(const char* name, F kern, int threads) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int smems[] = {100 * 1024, 200 * 1024, 227 * 1024};
  for (int smem : smems) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    printf("%s threads %d smem %d KB:", name, threads, smem / 1024);
    for (int cl = 1; cl <= 16; ++cl) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cl * 64);
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
      if (e != cudaSuccess) { cudaGetLastError(); n = -1; }
      printf(" %d:%d(%d)", cl, n, n * cl);
    }
    printf("\n");
  }
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("%s SMs %d\n", p.name, p.multiProcessorCount);
  probe("k256", k256, 256);
  probe("k512", k512, 512);
  return 0;
}
