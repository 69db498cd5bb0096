// Microbenchmarks for the roofline denominators of the Kaczmarz kernels on B200:
//   * shared-memory delivery bandwidth (bytes delivered to threads per cycle per SM)
//     for broadcast LDS.128 (every lane the same address), lane-distinct LDS.128
//     and LDS.64, which is what the lockstep kernels stream their rows with;
//   * FP32 FFMA throughput per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int THREADS = 512;
constexpr int ITERS = 4096;

template <int MODE>
__global__ void __launch_bounds__(THREADS) smem_kernel(float* out, long long* cyc) {
  __shared__ __align__(16) float4 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
    int base = (it * 16 + w * 64) & 2047;
    if (MODE == 0) {  // broadcast LDS.128
      float4 v = buf[(base + (it & 7)) & 2047];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    } else if (MODE == 1) {  // lane-distinct LDS.128
      float4 v = buf[(base + lane) & 2047];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    } else {  // lane-distinct LDS.64
      float2 v = reinterpret_cast<float2*>(buf)[(2 * base + lane) & 4095];
      acc.x += v.x; acc.y += v.y;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

__global__ void __launch_bounds__(THREADS) fma_kernel(float* out, long long* cyc, float a) {
  float r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = threadIdx.x * 0.001f + k;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = fmaf(r[k], a, 0.5f);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += r[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(float) * sms * THREADS * 2);
  cudaMalloc(&cyc, sizeof(long long) * sms * 2);
  long long h[4096];
  const char* names[3] = {"LDS.128 broadcast", "LDS.128 distinct", "LDS.64 distinct"};
  const int bytes_per_lane[3] = {16, 16, 8};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      if (mode == 0) smem_kernel<0><<<sms, THREADS>>>(out, cyc);
      if (mode == 1) smem_kernel<1><<<sms, THREADS>>>(out, cyc);
      if (mode == 2) smem_kernel<2><<<sms, THREADS>>>(out, cyc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
      double mc = 0;
      for (int s = 0; s < sms; ++s) mc += h[s];
      mc /= sms;
      double bytes_sm = (double)THREADS * ITERS * bytes_per_lane[mode];
      if (rep == 1)
        printf("{\"probe\": \"%s\", \"bytes_per_cycle_per_sm\": %.1f, \"chip_TBps\": %.2f, \"ms\": %.3f}\n",
               names[mode], bytes_sm / mc, bytes_sm * sms / (ms * 1e-3) / 1e12, ms);
    }
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    fma_kernel<<<sms * 2, THREADS>>>(out, cyc, 0.999f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(h, cyc, sizeof(long long) * sms * 2, cudaMemcpyDeviceToHost);
    double mc = 0;
    for (int s = 0; s < sms * 2; ++s) mc += h[s];
    mc /= sms * 2;
    double fma_sm = 2.0 * THREADS * ITERS * 8;  // two resident CTAs per SM
    if (rep == 1)
      printf("{\"probe\": \"FFMA\", \"fma_per_cycle_per_sm\": %.1f, \"chip_TFLOPs_fp32\": %.2f, \"ms\": %.3f}\n",
             fma_sm / mc, 2.0 * THREADS * ITERS * 8 * sms * 2 / (ms * 1e-3) / 1e12, ms);
  }
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
  return 0;
}
