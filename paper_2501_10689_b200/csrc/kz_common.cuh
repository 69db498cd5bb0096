// Common device helpers for the batched Kaczmarz kernels (sm_100a).
//
// Complex values are interleaved (re, im) pairs: float2 for complex64 and
// double2 for complex128.  Arithmetic follows the reference's numpy semantics
// where it matters for row selection:
//   * |z| as numpy's SIMD cabs: sqrt(fma(lo/hi, lo/hi, 1)) * hi
//   * float64 sums of greedy weights as numpy's 8-accumulator pairwise sum
//   * Generator.choice as searchsorted(cumsum(p)/cumsum(p)[-1], u, 'right')
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/kaczmarz_b200.h"

// Optional per-phase cycle accounting (build variant `timing`, -DKZ_TIMING):
// thread 0 of each CTA accumulates clock64() deltas between CTA barriers.
#ifdef KZ_TIMING
// per CTA dump: [0..9] phase cycles (0 = setup, k = segment ending at the k-th CTA barrier of an
// iteration), [10] wall ns, [11] smid, [12..43] per-warp cycles from iteration start to the end of
// the warp's refresh (KZ_WSTAMP), summed over iterations.
#define KZ_TSTART __shared__ volatile int kz_dummy; long long kz_t_last = clock64(); long long kz_ph[12] = {0}; \
  long long kz_sm[8] = {0}; const long long kz_s0 = kz_t_last; \
  int kz_pi = 0; long long kz_w0 = 0, kz_wacc = 0; \
  unsigned long long kz_g0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(kz_g0));
#define KZ_PHASE() do { (void)kz_dummy; if (threadIdx.x == 0) { long long n_ = clock64(); \
  kz_ph[kz_pi < 9 ? kz_pi : 9] += n_ - kz_t_last; kz_t_last = n_; } ++kz_pi; } while (0)
#define KZ_ITER() (kz_pi = 1, kz_w0 = clock64())
// setup checkpoint k (< 8): cycles since kernel start on thread 0, dumped to slots [36 + k] (kernels with at
// most 24 warps, whose per-warp slots stop below 36)
#define KZ_SETUP_MARK(k) do { if (threadIdx.x == 0) kz_sm[(k) & 7] = clock64() - kz_s0; } while (0)
#define KZ_WSTAMP() (kz_wacc += clock64() - kz_w0)
// per-warp arrival time at one chosen point of the iteration (-DKZ_WSTAMP_AT=k picks the point k)
#ifndef KZ_WSTAMP_AT
#define KZ_WSTAMP_AT 0
#endif
#define KZ_WSTAMP_IF(k) do { if (KZ_WSTAMP_AT == (k)) KZ_WSTAMP(); } while (0)
#define KZ_TDUMP(ptr) do { if ((ptr)) { long long* o_ = (ptr) + (size_t)blockIdx.x * 44; \
  if ((threadIdx.x & 31) == 0 && (threadIdx.x >> 5) < 24) o_[12 + (threadIdx.x >> 5)] = kz_wacc; \
  if (threadIdx.x == 0 && blockDim.x <= 768) for (int q_ = 0; q_ < 8; ++q_) o_[36 + q_] = kz_sm[q_]; \
  if (threadIdx.x == 0) { unsigned long long g1_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1_)); \
  kz_ph[10] = (long long)(g1_ - kz_g0); unsigned smid_; asm("mov.u32 %0, %%smid;" : "=r"(smid_)); kz_ph[11] = smid_; \
  for (int q_ = 0; q_ < 12; ++q_) o_[q_] = kz_ph[q_]; } } } while (0)
#else
#define KZ_TSTART
#define KZ_PHASE() do {} while (0)
#define KZ_ITER() ((void)0)
#define KZ_SETUP_MARK(k) do {} while (0)
#define KZ_WSTAMP() ((void)0)
#define KZ_WSTAMP_IF(k) do {} while (0)
#define KZ_TDUMP(ptr) do {} while (0)
#endif

// Bounds-checked build variant `checked` (-DKZ_CHECKED, python -m paper_2501_10689_b200.build --checked): the
// shared-memory, cluster-shared-memory (DSMEM), TMEM and piece-list indices the on-chip kernels compute are checked
// against their allocations; a violation prints the site and traps.  It stands in for compute-sanitizer memcheck,
// which is closed on this GPU pool (tools/sanitize_cases.py runs every kernel under it).
#ifdef KZ_CHECKED
#include <cstdio>
#define KZ_CHECK(cond, what)                                                                                        \
  do {                                                                                                            \
    if (!(cond)) {                                                                                                \
      printf("[kz checked] %s:%d: %s violated (block %d thread %d)\n", __FILE__, __LINE__, what, (int)blockIdx.x,  \
             (int)threadIdx.x);                                                                                   \
      __trap();                                                                                                   \
    }                                                                                                             \
  } while (0)
#else
#define KZ_CHECK(cond, what) do {} while (0)
#endif

namespace kz {

constexpr unsigned FULL = 0xffffffffu;

// host side: set by kz_solve_workspace_bytes_for while it asks the dispatchers which kernel a call would take;
// every launch function returns 1 ("would launch") right before its kernel launch when it is set
inline thread_local bool g_dry_launch = false;

template <class T> struct Cx;
template <> struct Cx<float2> {
  using real = float;
  static __host__ __device__ __forceinline__ float2 make(float r, float i) { return make_float2(r, i); }
};
template <> struct Cx<double2> {
  using real = double;
  static __host__ __device__ __forceinline__ double2 make(double r, double i) { return make_double2(r, i); }
};

template <class T> __device__ __forceinline__ T cadd(T a, T b) { return Cx<T>::make(a.x + b.x, a.y + b.y); }
template <class T> __device__ __forceinline__ T csub(T a, T b) { return Cx<T>::make(a.x - b.x, a.y - b.y); }
// a * b
template <class T> __device__ __forceinline__ T cmul(T a, T b) {
  return Cx<T>::make(fma(a.x, b.x, -(a.y * b.y)), fma(a.x, b.y, a.y * b.x));
}
// acc += conj(a) * b
template <class T> __device__ __forceinline__ T cfma_conj(T a, T b, T acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
  return acc;
}
// acc += a * b
template <class T> __device__ __forceinline__ T cfma(T a, T b, T acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
// packed fp32x2 FMA (sm_100a FFMA2): d = a * b + c per half, one rounding per half (bitwise the same as two
// fmaf calls); a broadcast scalar operand (fma2s) is folded into the instruction by ptxas
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long A, B, C, D;
  asm("mov.b64 %0, {%1, %2};" : "=l"(A) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(B) : "f"(b.x), "f"(b.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(C) : "f"(c.x), "f"(c.y));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(D) : "l"(A), "l"(B), "l"(C));
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(D));
  return r;
}
__device__ __forceinline__ float2 fma2s(float s, float2 b, float2 c) { return fma2(make_float2(s, s), b, c); }
template <class T> __device__ __forceinline__ T cscale(T a, typename Cx<T>::real s) { return Cx<T>::make(a.x * s, a.y * s); }
template <class T> __device__ __forceinline__ T cdivr(T a, double e) {
  using R = typename Cx<T>::real;
  return Cx<T>::make(a.x / (R)e, a.y / (R)e);
}
template <class T> __device__ __forceinline__ double2 to_d2(T a) { return make_double2((double)a.x, (double)a.y); }
template <class T> __device__ __forceinline__ T from_d2(double2 a) {
  using R = typename Cx<T>::real;
  return Cx<T>::make((R)a.x, (R)a.y);
}
template <class T> __device__ __forceinline__ T czero() { return Cx<T>::make(0, 0); }

// asynchronous global -> shared copy of one 8-byte element (LDGSTS), zero-filled when !valid: the setup
// loops issue every row piece without waiting on each load (cp_async_wait_all + a barrier before use)
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc, bool valid) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(gsrc), "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// numpy SIMD complex abs (verified bit-exact against np.abs on AVX-512 hosts).
__device__ __forceinline__ double np_cabs(double re, double im) {
  double a = fabs(re), b = fabs(im);
  double hi = a > b ? a : b, lo = a > b ? b : a;
  if (hi == 0.0) return 0.0;
  double r = lo / hi;
  return sqrt(fma(r, r, 1.0)) * hi;
}
__device__ __forceinline__ double np_abs2(double re, double im) {
  double a = np_cabs(re, im);
  return a * a;
}

template <class R> __device__ __forceinline__ R warp_sum(R v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
template <class T> __device__ __forceinline__ T warp_csum(T v) {
  v.x = warp_sum(v.x);
  v.y = warp_sum(v.y);
  return v;
}

__device__ inline double np_pairwise_sum(const double* a, int n);
// numpy pairwise summation (umath loops, PW_BLOCKSIZE 128, 8-way unroll),
// evaluated by one thread.  Blocks above 128 split at n/2 rounded down to a
// multiple of 8, exactly as numpy does.
__device__ inline double np_pairwise_block(const double* a, int m) {
  if (m < 8) {
    double res = 0.0;
    for (int i = 0; i < m; ++i) res += a[i];
    return res;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int full = m - (m % 8);
  for (int i = 8; i < full; i += 8)
    for (int j = 0; j < 8; ++j) r[j] += a[i + j];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (int i = full; i < m; ++i) res += a[i];
  return res;
}
// the same sum with the warp: lanes 0..7 run the eight accumulator chains of a block (independent loads, the same
// additions in the same order), lane 0 combines them and adds the tail -- bitwise np_pairwise_block for n <= 128;
// result in every lane
__device__ inline double np_pairwise_sum_warp(const double* a, int n, int lane) {
  if (n > 128 || n < 8) {
    double t = 0.0;
    if (lane == 0) t = np_pairwise_sum(a, n);
    return __shfl_sync(FULL, t, 0);
  }
  const int full = n - (n % 8);
  double r = 0.0;
  if (lane < 8) {
    r = a[lane];
#pragma unroll 4
    for (int i = 8 + lane; i < full; i += 8) r += a[i];
  }
  double rr[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) rr[j] = __shfl_sync(FULL, r, j);
  double res = ((rr[0] + rr[1]) + (rr[2] + rr[3])) + ((rr[4] + rr[5]) + (rr[6] + rr[7]));
  for (int i = full; i < n; ++i) res += a[i];
  return res;
}
__device__ inline double np_pairwise_sum(const double* a, int n) {
  if (n <= 128) return np_pairwise_block(a, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
}

// ---------------------------------------------------------------- Philox4x32-10
struct U4 { uint32_t x, y, z, w; };
__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += W0;
    k1 += W1;
  }
  return c;
}
// uniform double in [0, 1) with 53 random bits, keyed by (seed, system, rhs, draw)
__device__ __forceinline__ double philox_uniform(uint64_t seed, uint32_t b, uint32_t rhs, uint64_t draw) {
  U4 c{(uint32_t)draw, (uint32_t)(draw >> 32), rhs, b};
  U4 o = philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  uint64_t bits = ((uint64_t)o.x << 32 | o.y) >> 11;
  return (double)bits * (1.0 / 9007199254740992.0);
}

// ---------------------------------------------------------------------------------------------------------------
// NMSE-stopped lockstep runs (run_precoding, solvers.py:583-603) on the on-chip kernels: the CTAs of one system form
// a thread-block cluster (at most NMX_MAX), reduce fixed-order fp64 partials per CTA and push them to every CTA of
// the cluster over DSMEM; every CTA sums the slots in rank order, so all of them take the same stop decision.
// Slots: [2][NMX_MAX] ||M||^2, [NMX_MAX] ||F_ref - F_now||^2, [2][NMX_MAX] flop sums, [2][NMX_MAX] done counts (the
// first exchange of an iteration alternates between two buffers by iteration parity, so a fast CTA's next push
// cannot overwrite slots a slow CTA still reads; the second exchange is ordered by the first of the next iteration)
constexpr int NMX_MAX = 8;
__host__ __device__ inline size_t nmx_bytes() { return (size_t)NMX_MAX * (16 + 8 + 16 + 8); }
struct NmxSlots {
  double* C;
  double* S;
  long long* F;
  int* D;
};
__device__ __forceinline__ NmxSlots nmx_slots(unsigned char* base) {
  NmxSlots x;
  x.C = (double*)base;
  x.S = x.C + 2 * NMX_MAX;
  x.F = (long long*)(x.S + NMX_MAX);
  x.D = (int*)(x.F + 2 * NMX_MAX);
  return x;
}
__device__ __forceinline__ uint32_t dsm_addr(const void* p, int rank) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void dsm_st(double* p, int rank, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(dsm_addr(p, rank)), "d"(v) : "memory");
}
__device__ __forceinline__ void dsm_st(long long* p, int rank, long long v) {
  asm volatile("st.shared::cluster.s64 [%0], %1;" ::"r"(dsm_addr(p, rank)), "l"(v) : "memory");
}
__device__ __forceinline__ void dsm_st(int* p, int rank, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(dsm_addr(p, rank)), "r"(v) : "memory");
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// fixed-order CTA sum of a double (warp tree, then the warp partials in warp order): identical in every thread
__device__ __forceinline__ double cta_sum_d(double v, double* red, int w, int lane, int nw) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int q = 0; q < nw; ++q) s += red[q];
  __syncthreads();  // red is rewritten by the next sum
  return s;
}
// first exchange of iteration t: the CTA's ||M||^2 (cs, every thread), done count and flop sum (nd, fs: threads
// tid < nct) -> the system's totals in every thread
__device__ __forceinline__ void nmx_round1(const NmxSlots& x, int t, int rank, int nct, int tid, double cs, int nd,
                                           long long fs, double& C, int& ndt, long long& fst) {
  const int o = NMX_MAX * (t & 1);
  if (tid < nct) {
    dsm_st(x.C + o + rank, tid, cs);
    dsm_st(x.D + o + rank, tid, nd);
    dsm_st(x.F + o + rank, tid, fs);
  }
  cluster_barrier();
  C = 0.0;
  ndt = 0;
  fst = 0;
  for (int r = 0; r < nct; ++r) {
    C += x.C[o + r];
    ndt += x.D[o + r];
    fst += x.F[o + r];
  }
}
// second exchange: the CTA's ||F_ref - F_now||^2 -> the system's total
__device__ __forceinline__ double nmx_round2(const NmxSlots& x, int rank, int nct, int tid, double ds) {
  if (tid < nct) dsm_st(x.S + rank, tid, ds);
  cluster_barrier();
  double S2 = 0.0;
  for (int r = 0; r < nct; ++r) S2 += x.S[r];
  return S2;
}

}  // namespace kz
