#include <cstdio>
#include <dlfcn.h>
#include <vector>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
__global__ void k2d(const __grid_constant__ CUtensorMap tmap, float* out, int x, int y) {
  __shared__ alignas(128) float buf[32 * 8];
  __shared__ alignas(8) unsigned long long bar;
  unsigned sb = (unsigned)__cvta_generic_to_shared(&bar), sd = (unsigned)__cvta_generic_to_shared(buf);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sb));
    asm volatile("fence.proxy.async.shared::cta;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sb), "r"(32 * 8 * 4));
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 :: "r"(sd), "l"(&tmap), "r"(x), "r"(y), "r"(sb) : "memory");
  }
  unsigned done = 0;
  while (!done) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }" : "=r"(done) : "r"(sb));
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = buf[i];
}
int main() {
  const int W = 256, H = 64;
  std::vector<float> h(W * H);
  for (int i = 0; i < W * H; ++i) h[i] = i;
  float *d, *o; cudaMalloc(&d, W * H * 4); cudaMalloc(&o, 256 * 4);
  cudaMemcpy(d, h.data(), W * H * 4, cudaMemcpyHostToDevice);
  void* fp = nullptr; cudaDriverEntryPointQueryResult q;
  void* lib = dlopen("libcuda.so.1", RTLD_NOW);
  void* fd = lib ? dlsym(lib, "cuTensorMapEncodeTiled") : nullptr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  printf("entry %p dlsym %p same %d\n", fp, fd, fp == fd);
  int drv = 0, rt = 0; cudaDriverGetVersion(&drv); cudaRuntimeGetVersion(&rt); printf("driver %d runtime %d\n", drv, rt);
  if (getenv("USE_DLSYM")) fp = fd;
  auto fn = (PFN_cuTensorMapEncodeTiled_v12000)fp;
  CUtensorMap m;
  cuuint64_t dim[2] = {W, H}; cuuint64_t st[1] = {W * 4}; cuuint32_t box[2] = {32, 8}; cuuint32_t es[2] = {1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dim, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  k2d<<<1, 32>>>(m, o, 5, 3);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> out(256); cudaMemcpy(out.data(), o, 1024, cudaMemcpyDeviceToHost);
  int bad = 0; for (int j = 0; j < 8; ++j) for (int i = 0; i < 32; ++i) if (out[j * 32 + i] != h[(3 + j) * W + 5 + i]) ++bad;
  printf("sync %s bad %d\n", cudaGetErrorString(e), bad);
}
