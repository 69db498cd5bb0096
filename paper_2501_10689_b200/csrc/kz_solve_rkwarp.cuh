// Warp-per-rhs kernel for the one-row-per-iteration schemes (urk, swor-erk) in complex64 or complex128, fixed T,
// contiguous VRs (solvers.py:382-389 with rk_step, solvers.py:173-188).
//
// An RK iteration touches one row (|Gamma_i| antennas) per rhs, so the wide kernel's CTA-wide barriers
// (draw -> partials -> step -> projection) dominate its time.  Here each warp owns one rhs and runs its T
// iterations without any CTA barrier: the iterate m of its rhs lives in shared memory (Nt complex), the
// rows of the system are shared by the warps of the CTA (packed, unpadded).  Per iteration the lanes
// stride the row's support (antenna s + lane + 32 j): one conflict-free LDS.64 of h and of m per element,
// a shuffle reduction for h^H m, the step, and the m update from the same registers.
#pragma once

#include "kz_common.cuh"
#include "kz_solve_generic.cuh"

namespace kz {

namespace rkw {

struct Plan {
  size_t rowS, rowL, hoff, en, M, Q, pool, total;
};

__host__ __device__ inline size_t al(size_t x) { return (x + 15) & ~size_t(15); }

// nw warps (rhs) per CTA, hcap packed H elements, cs bytes per complex (8: complex64, 16: complex128)
__host__ __device__ inline Plan plan(int K, int Nt, int nw, int hcap, int cs = 8) {
  Plan p;
  const int KW = (K + 31) / 32;
  size_t o = 0;
  p.rowS = o; o = al(o + 4 * (size_t)K);
  p.rowL = o; o = al(o + 4 * (size_t)K);
  p.hoff = o; o = al(o + 4 * (size_t)K);
  p.en = o; o = al(o + 8 * (size_t)K);
  p.M = o; o = al(o + (size_t)cs * nw * Nt);
  p.Q = o; o = al(o + (size_t)cs * nw * K);
  p.pool = o; o = al(o + 4 * (size_t)nw * KW);
  o = al(o + (size_t)cs * hcap);  // H last
  p.total = o;
  return p;
}

}  // namespace rkw

// T = float2 (throughput) or double2 (oracle mode: numpy's complex scalar x array products)
template <int SCH, class T>
__global__ void __launch_bounds__(1024, 1) kz_rkwarp_kernel(LsArgs p, int nw) {
  using namespace rkw;
  using Rl = typename Cx<T>::real;
  constexpr bool EXACT = sizeof(T) == 16;
  extern __shared__ __align__(16) unsigned char sm[];
  const int K = p.P.n_users, Nt = p.P.n_antennas;
  const int ngroups = (K + nw - 1) / nw;
  const int b = blockIdx.x / ngroups, c0g = (blockIdx.x % ngroups) * nw;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31, nthr = blockDim.x;
  const int KW = (K + 31) / 32;
  const Plan pl = plan(K, Nt, nw, p.hcap, (int)sizeof(T));
  int* rowS = (int*)(sm + pl.rowS);
  int* rowL = (int*)(sm + pl.rowL);
  int* hoff = (int*)(sm + pl.hoff);
  double* en = (double*)(sm + pl.en);
  T* Ms = (T*)(sm + pl.M) + (size_t)w * Nt;
  T* Qs = (T*)(sm + pl.Q) + (size_t)w * K;
  uint32_t* pool = (uint32_t*)(sm + pl.pool) + (size_t)w * KW;
  T* Hs = (T*)(sm + pl.pool + al(4 * (size_t)nw * KW));
  const Rl regf = (Rl)p.P.reg[b];

  for (int i = tid; i < K; i += nthr) {
    const size_t r = (size_t)b * K + i;
    const int sg = p.P.row_seg_ptr[r];
    rowS[i] = p.P.seg_start[sg];
    rowL[i] = p.P.seg_len[sg];
    en[i] = p.P.row_energy[r];
  }
  __syncthreads();
  if (w == 0) {  // packed row offsets
    int carry = 0;
    for (int base = 0; base < K; base += 32) {
      const int i = base + lane;
      const int v = i < K ? rowL[i] : 0;
      int sc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t2 = __shfl_up_sync(FULL, sc, o);
        if (lane >= o) sc += t2;
      }
      if (i < K) hoff[i] = carry + sc - v;
      carry += __shfl_sync(FULL, sc, 31);
    }
  }
  __syncthreads();
  {
    const T* heff = (const T*)p.P.heff;
    for (int i = w; i < K; i += nthr >> 5) {
      const T* src = heff + p.P.row_val_ptr[(size_t)b * K + i];
      for (int e = lane; e < rowL[i]; e += 32) {  // no wait per row
        if constexpr (EXACT) {
          const uint32_t d = (uint32_t)__cvta_generic_to_shared(Hs + hoff[i] + e);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + e) : "memory");
        } else {
          cp_async8(Hs + hoff[i] + e, src + e, true);
        }
      }
    }
    cp_async_wait_all();
  }
  for (int n = lane; n < Nt; n += 32) Ms[n] = czero<T>();
  for (int i = lane; i < K; i += 32) Qs[i] = czero<T>();
  for (int q = lane; q < KW; q += 32) pool[q] = 0;
  int poolcnt = 0;
  __syncthreads();

  const int c = c0g + w;
  const bool active = c < K && w < nw;
  long long flops = 0;
  int it = 0;
  if (active) {
    const size_t rid = (size_t)b * K + c;
    // draws in batches of 32: lane l evaluates (or loads) the draw of iteration it0 + l once, iteration it takes
    // it with a shuffle -- the same stream values, one Philox evaluation / one coalesced load per 32 iterations
    double ubuf = 0.0;
    int ibuf = 0;
    auto refill = [&](int it0) {
      const int d = it0 + lane;
      if (p.R.kind == KZ_RNG_HOST_INDEX) {
        if (d < p.T) ibuf = p.R.indices[rid * p.R.stream_len + d];
      } else if (p.R.kind == KZ_RNG_PHILOX) {
        ubuf = philox_uniform(p.R.seed, (uint32_t)(b + p.R.system_base), (uint32_t)c, (uint64_t)d);
      } else if (d < p.T) {
        ubuf = p.R.uniforms[rid * p.R.stream_len + d];
      }
    };
    for (it = 0; it < p.T; ++it) {
      if ((it & 31) == 0) refill(it);
      // ---- draw (solvers.py:218-230)
      int i;
      if (p.R.kind == KZ_RNG_HOST_INDEX) {
        i = __shfl_sync(FULL, ibuf, it & 31);
      } else if (SCH == KZ_URK) {
        const double u = __shfl_sync(FULL, ubuf, it & 31);
        i = (int)(u * K);
        i = i >= K ? K - 1 : i;
      } else {  // energy-weighted pick without replacement from the epoch pool (warp-parallel scan)
        if (poolcnt == 0) {
          for (int q = lane; q < KW; q += 32) pool[q] = 0xFFFFFFFFu >> (q == KW - 1 && (K & 31) ? 32 - (K & 31) : 0);
          poolcnt = K;
          __syncwarp();
        }
        const double u = __shfl_sync(FULL, ubuf, it & 31);
        double tot = 0.0;
        for (int j = lane; j < K; j += 32)
          if ((pool[j >> 5] >> (j & 31)) & 1u) tot += en[j];
        tot = warp_sum(tot);
        const double tau = u * tot;
        double carry = 0.0;
        int pick = -1, last = -1;
        for (int base = 0; base < K; base += 32) {
          const int j = base + lane;
          const bool in = j < K && ((pool[j >> 5] >> (j & 31)) & 1u);
          const double v = in ? en[j] : 0.0;
          double sc = v;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const double t2 = __shfl_up_sync(FULL, sc, o);
            if (lane >= o) sc += t2;
          }
          const unsigned hit = __ballot_sync(FULL, in && carry + sc > tau);
          const unsigned nz = __ballot_sync(FULL, in);
          if (pick < 0 && hit) pick = base + __ffs(hit) - 1;
          if (nz) last = base + 31 - __clz(nz);
          carry += __shfl_sync(FULL, sc, 31);
        }
        i = pick >= 0 ? pick : last;
        __syncwarp();
        if (lane == 0) pool[i >> 5] &= ~(1u << (i & 31));
        __syncwarp();
        poolcnt -= 1;
      }
      if (SCH == KZ_SWOR_ERK) flops += (K - it % K) + 2;  // pool bookkeeping charge (as the wide kernel)
      // ---- refresh of row i (solvers.py:159-170) and rk_step (solvers.py:173-188)
      const int s = rowS[i], L = rowL[i];
      const T* h = Hs + hoff[i];
      Rl dx = 0, dy = 0;
      for (int e = lane; e < L; e += 32) {
        const T hv = h[e], mv = Ms[s + e];
        dx = fma(hv.x, mv.x, dx); dx = fma(hv.y, mv.y, dx);
        dy = fma(hv.x, mv.y, dy); dy = fma(-hv.y, mv.x, dy);
      }
      dx = warp_sum(dx);
      dy = warp_sum(dy);
      const T q = Qs[i];
      const Rl tg = i == c ? (Rl)1 : (Rl)0;
      const T r = Cx<T>::make((tg - dx) - q.x * regf, ((Rl)0 - dy) - q.y * regf);
      const Rl e = (Rl)en[i];
      const T gm = Cx<T>::make(r.x / e, r.y / e);
      for (int e2 = lane; e2 < L; e2 += 32) {
        const T hv = h[e2];
        T mv = Ms[s + e2];
        if constexpr (EXACT) {  // col[idx] += gamma * eff_rows[i] (numpy scalar x array, then add)
          mv = cadd(mv, cmul(gm, hv));
        } else {
          mv.x = fmaf(gm.x, hv.x, mv.x); mv.x = fmaf(-gm.y, hv.y, mv.x);
          mv.y = fmaf(gm.x, hv.y, mv.y); mv.y = fmaf(gm.y, hv.x, mv.y);
        }
        Ms[s + e2] = mv;
      }
      if (lane == 0) {
        Qs[i] = Cx<T>::make(q.x + gm.x, q.y + gm.y);
        if (p.O.rows && it < p.O.rows_cap) p.O.rows[rid * p.O.rows_cap + it] = i;
      }
      flops += 2 * (8LL * Nt + 4);
      __syncwarp();
    }
  }
  // ---- outputs
  if (active) {
    const size_t rid = (size_t)b * K + c;
    T* vout = (T*)p.O.v;
    for (int i = lane; i < K; i += 32) vout[((size_t)b * K + i) * K + c] = Qs[i];
    if (p.O.iterates) {
      T* M = (T*)p.O.iterates + rid * Nt;
      for (int n = lane; n < Nt; n += 32) M[n] = Ms[n];
    }
    if (lane == 0) {
      if (p.O.iters) p.O.iters[rid] = it;
      if (p.O.converged) p.O.converged[rid] = 0;
      if (p.O.done) p.O.done[rid] = 0;
      if (p.O.noop_steps) p.O.noop_steps[rid] = 0;
      if (p.O.flops) p.O.flops[rid] = flops;
    }
  }
  if (tid == 0) p.tstop[blockIdx.x] = p.T;
}

// 1 launched, 0 not eligible, -1 failure
inline int rkwarp_dispatch(const kz_problem& P, int scheme, const kz_rng& R, const kz_out& O, int T_iters, char* ws,
                           int32_t* tstop, int maxsm, cudaStream_t s) {
  if (scheme != KZ_URK && scheme != KZ_SWOR_ERK) return 0;
  if (!(P.flags & KZ_PROBLEM_CONTIGUOUS)) return 0;
  static const bool off = getenv("KZ_DISABLE_RKWARP") != nullptr;  // A/B switch
  if (off) return 0;
  const int K = P.n_users, Nt = P.n_antennas;
  const int hcap = K * P.max_support;
  int nw = K < 32 ? K : 32;
  size_t smem = 0;
  const int cs = P.dtype == KZ_C128 ? 16 : 8;
  for (; nw >= 1; nw = nw > 8 ? nw - 8 : nw - 1) {
    smem = rkw::plan(K, Nt, nw, hcap, cs).total;
    if (smem <= (size_t)maxsm) break;
  }
  if (nw < 1) return 0;
  LsArgs a;
  a.f_ref = nullptr;
  a.eps = 0.0;
  a.bulk = 0;
  a.P = P;
  a.R = R;
  a.O = O;
  a.T = T_iters;
  a.S = 0;
  a.hcap = hcap;
  a.ws = ws;
  a.L = gen_layout(P.n_systems, P.n_users, P.n_antennas, P.dtype);
  a.tstop = tstop;
  const int groups = (K + nw - 1) / nw;
  auto kern = P.dtype == KZ_C128
                  ? (scheme == KZ_URK ? kz_rkwarp_kernel<KZ_URK, double2> : kz_rkwarp_kernel<KZ_SWOR_ERK, double2>)
                  : (scheme == KZ_URK ? kz_rkwarp_kernel<KZ_URK, float2> : kz_rkwarp_kernel<KZ_SWOR_ERK, float2>);
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return -1;
  if (g_dry_launch) return 1;
  kern<<<P.n_systems * groups, 32 * nw, smem, s>>>(a, nw);
  kz_lockstep_finalize<<<(P.n_systems + 127) / 128, 128, 0, s>>>(tstop, groups, P.n_systems, O.n_outer,
                                                                  O.sys_converged);
  return 1;
}

}  // namespace kz
