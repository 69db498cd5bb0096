// FFMA issue-rate probes on B200 (sm_100a): which FMA instruction forms reach the FP32 pipe peak.
//   imm   : r = fmaf(r, a, 0.5f)            (immediate operand: 2 register reads)
//   reg3  : acc = fmaf(h, m, acc)           (3 register reads, h broadcast per pair of FMAs, m per FMA:
//                                            the refresh loop's pattern, conj(h) . m over register-resident m)
//   ffma2 : acc2 = fma(h2, m2, acc2) packed (FFMA2 on (x, y) pairs, 3 x 64-bit register reads)
//   ffma2s: acc2 = fma((h, h), m2, acc2)    (scalar broadcast operand folded into FFMA2)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fma_forms tools/fma_forms.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int THREADS = 512;
constexpr int ITERS = 2048;

__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
  unsigned long long d;
  const unsigned long long A = *reinterpret_cast<unsigned long long*>(&a), B = *reinterpret_cast<unsigned long long*>(&b),
                           C = *reinterpret_cast<unsigned long long*>(&c);
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(A), "l"(B), "l"(C));
  return *reinterpret_cast<float2*>(&d);
}

template <int MODE>
__global__ void __launch_bounds__(THREADS, 1) fma_kernel(float* out, long long* cyc, float a) {
  // 16 "iterate" registers (m) and 8 accumulators, like one 2-rhs dot product over 8 complex elements
  float m[16], acc[8];
#pragma unroll
  for (int k = 0; k < 16; ++k) m[k] = threadIdx.x * 0.001f + k;
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = 0.f;
  float h0 = a, h1 = a * 0.5f, h2 = a * 0.25f, h3 = a * 0.125f;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    if (MODE == 0) {
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = fmaf(acc[k], a, 0.5f);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = fmaf(acc[k], a, 0.5f);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = fmaf(acc[k], a, 0.5f);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = fmaf(acc[k], a, 0.5f);
    } else if (MODE == 1) {
      // 32 FMAs: 4 "h" scalars x 8 accumulators, each with its own m register
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = fmaf(h0, m[k], acc[k]);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = fmaf(h1, m[k + 8], acc[k]);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = fmaf(h2, m[(k + 4) & 15], acc[k]);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = fmaf(h3, m[(k + 12) & 15], acc[k]);
    } else if (MODE == 2) {
      // 16 FFMA2 = 32 FMAs: packed h pairs x packed m pairs
      float2* A2 = reinterpret_cast<float2*>(acc);
      const float2* M2 = reinterpret_cast<const float2*>(m);
      const float2 ha = make_float2(h0, h1), hb = make_float2(h2, h3);
#pragma unroll
      for (int k = 0; k < 4; ++k) A2[k] = f2fma(ha, M2[k], A2[k]);
#pragma unroll
      for (int k = 0; k < 4; ++k) A2[k] = f2fma(hb, M2[k + 4], A2[k]);
#pragma unroll
      for (int k = 0; k < 4; ++k) A2[k] = f2fma(ha, M2[(k + 2) & 7], A2[k]);
#pragma unroll
      for (int k = 0; k < 4; ++k) A2[k] = f2fma(hb, M2[(k + 6) & 7], A2[k]);
    } else {
      // 16 FFMA2 with a broadcast scalar (h, h)
      float2* A2 = reinterpret_cast<float2*>(acc);
      const float2* M2 = reinterpret_cast<const float2*>(m);
#pragma unroll
      for (int k = 0; k < 4; ++k) A2[k] = f2fma(make_float2(h0, h0), M2[k], A2[k]);
#pragma unroll
      for (int k = 0; k < 4; ++k) A2[k] = f2fma(make_float2(h1, h1), M2[k + 4], A2[k]);
#pragma unroll
      for (int k = 0; k < 4; ++k) A2[k] = f2fma(make_float2(h2, h2), M2[(k + 2) & 7], A2[k]);
#pragma unroll
      for (int k = 0; k < 4; ++k) A2[k] = f2fma(make_float2(h3, h3), M2[(k + 6) & 7], A2[k]);
    }
    h0 += 1e-7f;  // keep h live-varying (as the LDS-fed h of the real loop)
    h1 += 1e-7f;
    h2 += 1e-7f;
    h3 += 1e-7f;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(const char* name, int sms, float* out, long long* cyc) {
  long long h[1024];
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    fma_kernel<MODE><<<sms, THREADS>>>(out, cyc, 0.999f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double mc = 0;
    for (int s = 0; s < sms; ++s) mc += h[s];
    mc /= sms;
    const double fma_sm = (double)THREADS * ITERS * 32;  // 32 FMAs per thread per trip in every mode
    if (rep == 1)
      printf("{\"probe\": \"%s\", \"fma_per_cycle_per_sm\": %.1f, \"warp_fma_instr_per_cycle_per_smsp\": %.3f, "
             "\"chip_TFLOPs_fp32\": %.2f, \"ms\": %.3f}\n",
             name, fma_sm / mc, fma_sm / mc / 4 / 32 / (MODE >= 2 ? 2 : 1), 2.0 * fma_sm * sms / (ms * 1e-3) / 1e12,
             ms);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(float) * sms * THREADS);
  cudaMalloc(&cyc, sizeof(long long) * sms);
  run<0>("FFMA imm", sms, out, cyc);
  run<1>("FFMA reg3", sms, out, cyc);
  run<2>("FFMA2 reg3", sms, out, cyc);
  run<3>("FFMA2 broadcast", sms, out, cyc);
  return 0;
}
