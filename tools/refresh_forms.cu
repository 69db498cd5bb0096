// Refresh inner-loop forms on B200 (sm_100a): cycles per (row, chunk) piece per SM sub-partition for the register
// blockings a warp can use on one 32-antenna chunk of 32 right-hand sides, H rows in shared memory, 16 warps per
// SM (the wide kernel's occupancy), every warp streaming the same number of pieces:
//   form A  2 rhs x 16 antennas per thread (lane = (a: 2, g: 16))   8 LDS.128 + 128 FFMA + 1 exchange stage
//           -- the wide kernel's blocking: LDS pipe and FFMA issue balanced
//   form B  4 rhs x  8 antennas per thread (lane = (a: 4, g:  8))   4 LDS.128 + 128 FFMA + 2 exchange stages
//           -- half the shared-memory wavefronts per FFMA
// Each form ends a piece the way the kernel does: a transpose-reduce over the a-lanes (every lane keeps one rhs'
// partial) and one 8-byte store into a slot array.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o tools/refresh_forms tools/refresh_forms.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int THREADS = 512, NPIECE = 64, ROWS = 64, ROW_EL = 160 + 2, ITERS = 200;

template <int FORM>
__global__ void __launch_bounds__(THREADS, 1) refresh_kernel(float2* out, long long* cyc, const int* order, float seed) {
  extern __shared__ __align__(16) unsigned char sm[];
  float2* Hs = (float2*)sm;                          // ROWS rows of ROW_EL elements
  float2* Ps = Hs + ROWS * ROW_EL;                   // [NPIECE][32] per warp slot array (shared by the warps: timing only)
  int* ord = (int*)(Ps + NPIECE * 32);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  for (int e = tid; e < ROWS * ROW_EL; e += THREADS) Hs[e] = make_float2(1e-3f * (e % 97), -1e-3f * (e % 89));
  for (int e = tid; e < NPIECE; e += THREADS) ord[e] = order[e];
  __syncthreads();
  const float4* H4 = reinterpret_cast<const float4*>(Hs);
  float2 m[32];  // the thread's iterate: FORM A m[r * 16 + k] (2 rhs x 16), FORM B m[r * 8 + k] (4 rhs x 8)
#pragma unroll
  for (int k = 0; k < 32; ++k) m[k] = make_float2(seed + 0.01f * k + 1e-3f * tid, 0.5f * seed - 0.01f * k * seed + 2e-3f * tid);  // run-time values: no immediates
  long long t0 = clock64();
  float4 hreg[8];
  float2 accs = make_float2(0.f, 0.f);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll 8
    for (int q = 0; q < NPIECE; ++q) {
      if (FORM == 4 && (q & 7) == 0) {  // eight row elements per eight pieces: 1/8 of the loop's LDS traffic
#pragma unroll
        for (int j = 0; j < 8; ++j) hreg[j] = H4[(ord[q] * (ROW_EL / 2) + it + 2 * j + 16 * (threadIdx.x >> 9)) & 4095];
      }
      const int row = ord[q];
      const int h0 = row * ROW_EL + 32 * ((w + q) & 3);  // a chunk of the row (element offset, even)
      if (FORM == 5) {
        // form A's blocking with packed FFMA2 (fma.rn.f32x2): the iterate of the two rhs planar, MX[k] = (m0[k].x, m1[k].x),
        // MY[k] = (m0[k].y, m1[k].y) (here: m[k] and m[16 + k] reinterpreted), h components broadcast to pairs;
        // RE += (hx,hx) MX + (hy,hy) MY, IM += (hx,hx) MY, IN += (hy,hy) MX (IM - IN at the end); two accumulator sets
        const int a = lane >> 4;
        const float4* hp = H4 + ((h0 + 2 * a) >> 1);
        unsigned long long re0 = 0, im0 = 0, in0 = 0, re1 = 0, im1 = 0, in1 = 0;
        const unsigned long long* MX = reinterpret_cast<const unsigned long long*>(m);       // 16 pairs
        const unsigned long long* MY = reinterpret_cast<const unsigned long long*>(m + 16);  // 16 pairs
#define KZ_F2(acc, hh, mm) asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(hh), "l"(mm))
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 h = hp[2 * j];
          const int k = 2 * j;
          unsigned long long hxx, hyy, hzz, hww;
          asm("mov.b64 %0, {%1, %1};" : "=l"(hxx) : "f"(h.x));
          asm("mov.b64 %0, {%1, %1};" : "=l"(hyy) : "f"(h.y));
          asm("mov.b64 %0, {%1, %1};" : "=l"(hzz) : "f"(h.z));
          asm("mov.b64 %0, {%1, %1};" : "=l"(hww) : "f"(h.w));
          KZ_F2(re0, hxx, MX[k]); KZ_F2(im0, hxx, MY[k]); KZ_F2(in0, hyy, MX[k]); KZ_F2(re0, hyy, MY[k]);
          KZ_F2(re1, hzz, MX[k + 1]); KZ_F2(im1, hzz, MY[k + 1]); KZ_F2(in1, hww, MX[k + 1]); KZ_F2(re1, hww, MY[k + 1]);
        }
#undef KZ_F2
        float2 r0 = *reinterpret_cast<float2*>(&re0), r1 = *reinterpret_cast<float2*>(&re1);
        float2 i0 = *reinterpret_cast<float2*>(&im0), i1 = *reinterpret_cast<float2*>(&im1);
        float2 n0 = *reinterpret_cast<float2*>(&in0), n1 = *reinterpret_cast<float2*>(&in1);
        const float px = r0.x + r1.x, py = (i0.x + i1.x) - (n0.x + n1.x), qx = r0.y + r1.y, qy = (i0.y + i1.y) - (n0.y + n1.y);
        const float sx = a ? px : qx, sy = a ? py : qy;
        const float rx = __shfl_xor_sync(0xffffffffu, sx, 16), ry = __shfl_xor_sync(0xffffffffu, sy, 16);
        Ps[q * 32 + lane] = a ? make_float2(qx + rx, qy + ry) : make_float2(px + rx, py + ry);
      } else if (FORM == 4) {
        // form A's FFMAs alone: h stays in registers (loaded once per outer iteration), no exchange, no store
        const int a = lane >> 4;
        float x0 = 0, y0 = 0, x1 = 0, y1 = 0, u0 = 0, v0 = 0, u1 = 0, v1 = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 h = hreg[(j + q) & 7];  // a different row element per piece: nothing is loop invariant
          const int k = 2 * j;
          x0 = fmaf(h.x, m[k].x, x0); x0 = fmaf(h.y, m[k].y, x0);
          y0 = fmaf(h.x, m[k].y, y0); y0 = fmaf(-h.y, m[k].x, y0);
          x1 = fmaf(h.z, m[k + 1].x, x1); x1 = fmaf(h.w, m[k + 1].y, x1);
          y1 = fmaf(h.z, m[k + 1].y, y1); y1 = fmaf(-h.w, m[k + 1].x, y1);
          u0 = fmaf(h.x, m[16 + k].x, u0); u0 = fmaf(h.y, m[16 + k].y, u0);
          v0 = fmaf(h.x, m[16 + k].y, v0); v0 = fmaf(-h.y, m[16 + k].x, v0);
          u1 = fmaf(h.z, m[17 + k].x, u1); u1 = fmaf(h.w, m[17 + k].y, u1);
          v1 = fmaf(h.z, m[17 + k].y, v1); v1 = fmaf(-h.w, m[17 + k].x, v1);
        }
        accs.x += (x0 + x1) + (u0 + u1) + (float)a;
        accs.y += (y0 + y1) + (v0 + v1);
      } else if (FORM == 0) {
        const int a = lane >> 4;
        const float4* hp = H4 + ((h0 + 2 * a) >> 1);
        float x0 = 0, y0 = 0, x1 = 0, y1 = 0, u0 = 0, v0 = 0, u1 = 0, v1 = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 h = hp[2 * j];
          const int k = 2 * j;
          x0 = fmaf(h.x, m[k].x, x0); x0 = fmaf(h.y, m[k].y, x0);
          y0 = fmaf(h.x, m[k].y, y0); y0 = fmaf(-h.y, m[k].x, y0);
          x1 = fmaf(h.z, m[k + 1].x, x1); x1 = fmaf(h.w, m[k + 1].y, x1);
          y1 = fmaf(h.z, m[k + 1].y, y1); y1 = fmaf(-h.w, m[k + 1].x, y1);
          u0 = fmaf(h.x, m[16 + k].x, u0); u0 = fmaf(h.y, m[16 + k].y, u0);
          v0 = fmaf(h.x, m[16 + k].y, v0); v0 = fmaf(-h.y, m[16 + k].x, v0);
          u1 = fmaf(h.z, m[17 + k].x, u1); u1 = fmaf(h.w, m[17 + k].y, u1);
          v1 = fmaf(h.z, m[17 + k].y, v1); v1 = fmaf(-h.w, m[17 + k].x, v1);
        }
        const float px = x0 + x1, py = y0 + y1, qx = u0 + u1, qy = v0 + v1;
        const float sx = a ? px : qx, sy = a ? py : qy;
        const float rx = __shfl_xor_sync(0xffffffffu, sx, 16), ry = __shfl_xor_sync(0xffffffffu, sy, 16);
        Ps[q * 32 + lane] = a ? make_float2(qx + rx, qy + ry) : make_float2(px + rx, py + ry);
      } else if (FORM == 2 || FORM == 3) {
        // form A's blocking with the FFMAs of one h element ordered so that each shares one multiplicand with its
        // predecessor (m.x h.x, m.x h.y, m.y h.y, m.y h.x, ...): one new register operand per FFMA
        const int a = lane >> 4;
        const float4* hp = H4 + ((h0 + 2 * a) >> 1);
        float x0 = 0, y0 = 0, x1 = 0, y1 = 0, u0 = 0, v0 = 0, u1 = 0, v1 = 0;
        float xa = 0, ya = 0, xb = 0, yb = 0, ua = 0, va = 0, ub = 0, vb = 0;
#define KZ_F(acc, p, q) do { if (FORM == 3) asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(acc) : "f"(p), "f"(q)); else acc = fmaf(p, q, acc); } while (0)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 h = hp[2 * j];
          const int k = 2 * j;
          const float nhy = -h.y, nhw = -h.w;
          KZ_F(x0, m[k].x, h.x); KZ_F(y0, m[k].x, nhy); KZ_F(xa, m[k].y, h.y); KZ_F(ya, m[k].y, h.x);
          KZ_F(va, m[16 + k].y, h.x); KZ_F(ua, m[16 + k].y, h.y); KZ_F(v0, m[16 + k].x, nhy); KZ_F(u0, m[16 + k].x, h.x);
          KZ_F(x1, m[k + 1].x, h.z); KZ_F(y1, m[k + 1].x, nhw); KZ_F(xb, m[k + 1].y, h.w); KZ_F(yb, m[k + 1].y, h.z);
          KZ_F(vb, m[17 + k].y, h.z); KZ_F(ub, m[17 + k].y, h.w); KZ_F(v1, m[17 + k].x, nhw); KZ_F(u1, m[17 + k].x, h.z);
        }
#undef KZ_F
        const float px = (x0 + xa) + (x1 + xb), py = (y0 + ya) + (y1 + yb), qx = (u0 + ua) + (u1 + ub), qy = (v0 + va) + (v1 + vb);
        const float sx = a ? px : qx, sy = a ? py : qy;
        const float rx = __shfl_xor_sync(0xffffffffu, sx, 16), ry = __shfl_xor_sync(0xffffffffu, sy, 16);
        Ps[q * 32 + lane] = a ? make_float2(qx + rx, qy + ry) : make_float2(px + rx, py + ry);
      } else {
        const int a = lane >> 3;
        const float4* hp = H4 + ((h0 + 2 * a) >> 1);
        float ax[4] = {0, 0, 0, 0}, ay[4] = {0, 0, 0, 0}, bx[4] = {0, 0, 0, 0}, by[4] = {0, 0, 0, 0};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 h = hp[4 * j];
          const int k = 2 * j;
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            ax[r] = fmaf(h.x, m[8 * r + k].x, ax[r]); ax[r] = fmaf(h.y, m[8 * r + k].y, ax[r]);
            ay[r] = fmaf(h.x, m[8 * r + k].y, ay[r]); ay[r] = fmaf(-h.y, m[8 * r + k].x, ay[r]);
            bx[r] = fmaf(h.z, m[8 * r + k + 1].x, bx[r]); bx[r] = fmaf(h.w, m[8 * r + k + 1].y, bx[r]);
            by[r] = fmaf(h.z, m[8 * r + k + 1].y, by[r]); by[r] = fmaf(-h.w, m[8 * r + k + 1].x, by[r]);
          }
        }
        float px[4], py[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) { px[r] = ax[r] + bx[r]; py[r] = ay[r] + by[r]; }
        // transpose-reduce over the four a-lanes: stage 1 (xor 16) keeps two rhs, stage 2 (xor 8) keeps one
        const bool hi = a & 2, lo = a & 1;
        const float s0x = hi ? px[0] : px[2], s0y = hi ? py[0] : py[2], s1x = hi ? px[1] : px[3], s1y = hi ? py[1] : py[3];
        const float k0x = (hi ? px[2] : px[0]) + __shfl_xor_sync(0xffffffffu, s0x, 16);
        const float k0y = (hi ? py[2] : py[0]) + __shfl_xor_sync(0xffffffffu, s0y, 16);
        const float k1x = (hi ? px[3] : px[1]) + __shfl_xor_sync(0xffffffffu, s1x, 16);
        const float k1y = (hi ? py[3] : py[1]) + __shfl_xor_sync(0xffffffffu, s1y, 16);
        const float tx = lo ? k0x : k1x, ty = lo ? k0y : k1y;
        const float fx = (lo ? k1x : k0x) + __shfl_xor_sync(0xffffffffu, tx, 8);
        const float fy = (lo ? k1y : k0y) + __shfl_xor_sync(0xffffffffu, ty, 8);
        Ps[q * 32 + lane] = make_float2(fx, fy);
      }
    }
    m[0].x += 1e-6f;  // keep the iterate live-varying
    m[17].y -= 1e-6f;
  }
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
  float2 s = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < 32; ++k) { s.x += m[k].x; s.y += m[k].y; }
  s.x += Ps[lane].x + accs.x + accs.y;
  out[blockIdx.x * THREADS + tid] = s;
}

template <int FORM>
void run(const char* name, int sms, float2* out, long long* cyc, const int* order) {
  const size_t smem = (size_t)ROWS * ROW_EL * 8 + (size_t)NPIECE * 32 * 8 + NPIECE * 4;
  cudaFuncSetAttribute(refresh_kernel<FORM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  long long h[1024];
  for (int rep = 0; rep < 2; ++rep) {
    refresh_kernel<FORM><<<sms, THREADS, smem>>>(out, cyc, order, 1.0f + 1e-3f * rep);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double mc = 0;
    for (int s = 0; s < sms; ++s) mc += h[s];
    mc /= sms;
    // 16 warps = 4 per sub-partition, each NPIECE * ITERS pieces
    const double per_piece_smsp = mc / (4.0 * NPIECE * ITERS);
    if (rep == 1)
      printf("{\"form\": \"%s\", \"cycles_per_piece_per_smsp\": %.1f, \"ffma_per_clk_per_smsp\": %.3f, \"err\": \"%s\"}\n", name,
             per_piece_smsp, 128.0 / per_piece_smsp, cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float2* out; long long* cyc; int* order;
  cudaMalloc(&out, sizeof(float2) * sms * THREADS);
  cudaMalloc(&cyc, sizeof(long long) * sms);
  cudaMalloc(&order, sizeof(int) * NPIECE);
  int ho[NPIECE];
  for (int q = 0; q < NPIECE; ++q) ho[q] = (q * 37) % ROWS;
  cudaMemcpy(order, ho, sizeof(ho), cudaMemcpyHostToDevice);
  run<0>("A: 2 rhs x 16 antennas per thread (wide kernel)", sms, out, cyc, order);
  run<1>("B: 4 rhs x 8 antennas per thread", sms, out, cyc, order);
  run<4>("E: form A, the 128 FFMAs alone (h in registers, no exchange / store)", sms, out, cyc, order);
  run<5>("F: form A with packed FFMA2 (planar iterate over the two rhs, 6 accumulator pairs)", sms, out, cyc, order);
  run<2>("C: form A, FFMAs ordered to share one multiplicand with the predecessor (16 accumulators)", sms, out, cyc, order);
  run<3>("D: form C with the FFMA order pinned (asm volatile)", sms, out, cyc, order);
  return 0;
}
