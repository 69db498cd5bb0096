// Microbenchmarks for the roofline denominators of the Kaczmarz kernels on B200 (run through
// tools/microbench.py, which samples the SM clock with nvidia-smi while they run and writes
// profiles/r02_microbench.json):
//   * FP32 FFMA throughput, chip-wide from CUDA events over long launches (~0.2 s each), for the three
//     instruction forms the kernels could use: immediate operand (r = r * a + 0.5), three registers
//     (acc = h * m + acc: the refresh / aggregation loops' form, h reused by four consecutive FFMAs as in the
//     kernels) and packed fma.rn.f32x2 (FFMA2, three 64-bit register pairs);
//   * shared-memory delivery bandwidth for broadcast and lane-distinct LDS.128 / LDS.64.
// Every number is derived from event time and the work done, never from per-CTA clock64 windows (two
// co-resident CTAs do not start together, which inflated the round-1 per-clock FFMA figure).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int THREADS = 512;

__global__ void __launch_bounds__(THREADS) ffma_imm(float* out, float a, int iters) {
  float r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = threadIdx.x * 0.001f + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = fmaf(r[k], a, 0.5f);
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += r[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(THREADS) ffma_reg3(float* out, const float* in, int iters) {
  float h[4], m[4], acc[16];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    h[k] = in[(threadIdx.x + k) & 255];
    m[k] = in[(threadIdx.x + 7 * k + 3) & 255];
  }
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[4 * i + j] = fmaf(h[i], m[j], acc[4 * i + j]);
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ unsigned long long pk(float x, float y) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}

__global__ void __launch_bounds__(THREADS) ffma2_reg3(float* out, const float* in, int iters) {
  unsigned long long h[4], m[4], acc[8];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    h[k] = pk(in[(threadIdx.x + k) & 255], in[(threadIdx.x + k + 1) & 255]);
    m[k] = pk(in[(threadIdx.x + 7 * k + 3) & 255], in[(threadIdx.x + 5 * k) & 255]);
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = 0ull;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
        asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[2 * i + j]) : "l"(h[i]), "l"(m[j + 2 * (i & 1)]));
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float x, y;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(acc[k]));
    s += x + y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
__global__ void __launch_bounds__(THREADS) smem_kernel(float* out, int iters) {
  __shared__ __align__(16) float4 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
#pragma unroll 4
  for (int it = 0; it < iters; ++it) {
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
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

template <class F>
static float time_ms(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();  // warm-up
  cudaEventRecord(e0);
  launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4;  // 4 x 512 threads per SM (64 warps: full occupancy)
  float *out, *in;
  cudaMalloc(&out, sizeof(float) * blocks * THREADS);
  cudaMalloc(&in, sizeof(float) * 256);
  float hin[256];
  for (int i = 0; i < 256; ++i) hin[i] = 1.0f + i * 1e-4f;
  cudaMemcpy(in, hin, sizeof hin, cudaMemcpyHostToDevice);
  const double threads = (double)blocks * THREADS;
  {
    const int it = 1 << 15;
    float ms = time_ms([&] { ffma_imm<<<blocks, THREADS>>>(out, 0.999f, it); });
    printf("{\"probe\": \"FFMA imm\", \"ms\": %.3f, \"fma_per_s\": %.6e, \"sms\": %d}\n", ms,
           threads * it * 8 / (ms * 1e-3), sms);
  }
  {
    const int it = 1 << 14;
    float ms = time_ms([&] { ffma_reg3<<<blocks, THREADS>>>(out, in, it); });
    printf("{\"probe\": \"FFMA reg3\", \"ms\": %.3f, \"fma_per_s\": %.6e, \"sms\": %d}\n", ms,
           threads * it * 16 / (ms * 1e-3), sms);
  }
  {
    const int it = 1 << 14;
    float ms = time_ms([&] { ffma2_reg3<<<blocks, THREADS>>>(out, in, it); });
    printf("{\"probe\": \"FFMA2 reg3\", \"ms\": %.3f, \"fma_per_s\": %.6e, \"sms\": %d}\n", ms,
           threads * it * 16 / (ms * 1e-3), sms);
  }
  const char* names[3] = {"LDS.128 broadcast", "LDS.128", "LDS.64"};
  const int bytes_per_lane[3] = {16, 16, 8};
  for (int mode = 0; mode < 3; ++mode) {
    const int it = 1 << 21;
    float ms = time_ms([&] {
      if (mode == 0) smem_kernel<0><<<blocks, THREADS>>>(out, it);
      if (mode == 1) smem_kernel<1><<<blocks, THREADS>>>(out, it);
      if (mode == 2) smem_kernel<2><<<blocks, THREADS>>>(out, it);
    });
    printf("{\"probe\": \"%s\", \"ms\": %.3f, \"bytes_per_s\": %.6e, \"sms\": %d}\n", names[mode], ms,
           threads * it * bytes_per_lane[mode] / (ms * 1e-3), sms);
  }
  return 0;
}
