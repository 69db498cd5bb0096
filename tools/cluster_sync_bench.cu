// Cluster barrier round-trip cost on B200 (sm_100a): N back-to-back barrier.cluster.arrive.release +
// wait.acquire per CTA, for cluster sizes 2..16 and 256-thread CTAs (the cluster kernel's shape), with and
// without one remote DSMEM store per thread in flight before each barrier (release must drain it).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cluster_sync_bench tools/cluster_sync_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 2000;

template <bool STORE>
__global__ void __launch_bounds__(256, 1) sync_kernel(long long* out) {
  __shared__ float buf[256];
  unsigned rank, n;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(n));
  const unsigned peer = (rank + 1) % n;
  unsigned a = (unsigned)__cvta_generic_to_shared(buf + threadIdx.x), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(peer));
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) {
    if (STORE) asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(ra), "f"((float)i) : "memory");
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

template <bool STORE>
void run(int cl) {
  auto k = sync_kernel<STORE>;
  if (cl > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int grid = cl * 4;
  long long* d;
  cudaMalloc(&d, sizeof(long long) * grid);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, k, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[64];
  cudaMemcpy(h, d, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < grid; ++i) m += h[i];
  m /= grid;
  printf("{\"probe\": \"cluster barrier%s\", \"cluster\": %d, \"cycles_per_barrier\": %.0f, \"status\": \"%s\"}\n",
         STORE ? " after a DSMEM store" : "", cl, m / N, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int cl : {2, 4, 8, 16}) {
    run<false>(cl);
    run<true>(cl);
  }
  return 0;
}
