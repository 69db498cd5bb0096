// Wide register-resident lockstep kernel for the single-row (RK) family in
// complex64: urk, swor-erk, gk, grk, vr-ogrk (fixed T, contiguous VRs).
//
// One CTA = one system x 32 right-hand sides.  Lane (a, g), a = lane >> 4,
// g = lane & 15, owns the two rhs c = g0 + g and c + 16 (register blocking)
// on the 16 antennas 32w + 4j + 2a + e (j < 8, e < 2) of warp w's chunk, so
// thread (w, lane) keeps 2 x 16 iterate entries in 64 registers.  Rows live
// in shared memory zero-padded to whole 32-antenna chunks; a (row, chunk)
// product is 8 LDS.128 per thread feeding 128 FMAs (each h element reused for
// both rhs) with no predicates.  The two a-lanes exchange one partial each
// (one shuffle pair), then every lane stores its own rhs partial into the slot
// array P[i][slot][rhs] (slot = chunk - first chunk of the row), summed in a
// fixed order by the warp that selects for that rhs (deterministic).
// Why: shared memory delivers 128 B/clk/SM on B200 (tools/microbench.cu, a
// broadcast LDS.128 costs as much as a distinct one) and FFMA issues 128
// lanes/clk/SM, so one rhs per h element (8 B -> 4 FMA) caps the refresh at
// 50% of the FMA roofline; two rhs per element balance the two pipes.
// Semantics: InstanceRun.step for urk / swor-erk / gk / grk / vr-ogrk
// (solvers.py:382-406) with the FlopCounter charges of each primitive.
#pragma once

#include "kz_common.cuh"
#include "kz_solve_generic.cuh"
#include "kz_tmem.cuh"

// per-scheme switches (bit = kz_scheme), measured with same-box A/B runs (tools/ab3.sh)
#ifndef KZ_WIDE_HALF_MASK
#define KZ_WIDE_HALF_MASK ((1 << KZ_GK) | (1 << KZ_GRK) | (1 << KZ_VR_OGRK) | (1 << KZ_VR_OAHK))
#endif
#ifndef KZ_WIDE_NF
#define KZ_WIDE_NF 4  // whole-chunk refresh pieces in flight per warp (vr-oahk: 2)
#endif
#ifndef KZ_WIDE_PARW_MASK
#define KZ_WIDE_PARW_MASK (1 << KZ_VR_OAHK)
#endif

namespace kz {

namespace wide {

constexpr int G = 32;
constexpr int CH = 32;  // chunk = antennas per warp
template <int A, int B> struct JRange { static constexpr int lo = A, hi = B; };
constexpr int HSKEW = 2;  // spare H elements (one 16-byte unit) per row: consecutive rows start one bank group apart
// [row][rhs] arrays (P slots, Q, R) are XOR-swizzled on the rhs index so that
// both access directions (lanes over rhs: refresh / projection; lanes over
// rows: finalise / selection) are bank-conflict free.
__device__ __forceinline__ int xs(int i, int rhs) { return i * G + (rhs ^ (i & 15)); }

struct Plan {
  int K, W, SL, hcap;
  size_t rowS, rowL, c0, c1, hoff, en, inv_en, cost, cmask, inset, lptr, lst, optr, olst, nptr, nlst, H, P, Q, R, Phi, Dp, sel,
      gam, num, sp, nz, noop, done, iters, flops, prev, pool, poolcnt, misc, mbar, WP, lspl, ospl, nspl, nmx, red, total;
};

__host__ __device__ inline size_t al(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline Plan plan(int K, int Nt, int SL, int hcap) {
  Plan p;
  p.K = K;
  p.W = Nt / CH;
  p.SL = SL;
  p.hcap = hcap;
  const int KW = (K + 31) / 32;
  size_t o = 0;
  p.rowS = o; o = al(o + 4 * K);
  p.rowL = o; o = al(o + 4 * K);
  p.c0 = o; o = al(o + 4 * K);
  p.c1 = o; o = al(o + 4 * K);
  p.hoff = o; o = al(o + 4 * K);
  p.en = o; o = al(o + 4 * K);
  p.inv_en = o; o = al(o + 4 * K);
  p.cost = o; o = al(o + 8 * K);
  p.cmask = o; o = al(o + 4 * (size_t)K * KW);
  p.inset = o; o = al(o + K);
  p.lptr = o; o = al(o + 4 * (p.W + 1));
  p.lst = o; o = al(o + 8 * (size_t)K * SL);
  p.optr = o; o = al(o + 4 * (p.W + 1));
  p.olst = o; o = al(o + 8 * (size_t)K * SL);
  p.nptr = o; o = al(o + 4 * (p.W + 1));
  p.nlst = o; o = al(o + 8 * (size_t)K * SL);
  p.H = o; o = al(o + 8 * (size_t)hcap);
  p.P = o; o = al(o + 8 * (size_t)K * SL * G);
  p.Q = o; o = al(o + 8 * (size_t)K * G);
  p.R = o; o = al(o + 8 * (size_t)K * G);
  p.Phi = o; o = al(o + 8 * (size_t)K * G);
  p.Dp = o; o = al(o + 4 * (size_t)p.W * G);
  p.sel = o; o = al(o + 4 * G);
  p.gam = o; o = al(o + 8 * G);
  p.num = o; o = al(o + 8 * G);
  p.sp = o; o = al(o + 4 * G);
  p.nz = o; o = al(o + 4 * G);
  p.noop = o; o = al(o + 4 * G);
  p.done = o; o = al(o + 4 * G);
  p.iters = o; o = al(o + 4 * G);
  p.flops = o; o = al(o + 8 * G);
  p.prev = o; o = al(o + 4 * G);
  p.pool = o; o = al(o + 4 * (size_t)G * KW);
  p.poolcnt = o; o = al(o + 4 * G);
  p.misc = o; o = al(o + 32);
  p.mbar = o; o = al(o + 8);
  p.lspl = o; o = al(o + 8 * (size_t)p.W);
  p.ospl = o; o = al(o + 8 * (size_t)p.W);
  p.nspl = o; o = al(o + 8 * (size_t)p.W);
  // NMSE-stopped runs: the cluster exchange slots (kz_common.cuh nmx_*) and the CTA reduction scratch
  p.nmx = o; o = al(o + nmx_bytes());
  p.red = o; o = al(o + 8 * (size_t)p.W);
  // per-warp weight partials of the aggregation schemes ([warp][rhs]: num float2, ||phi||^2, nonzero flag); they
  // live in R (unused by AHK / VR-OAHK) when it is large enough
  if ((size_t)K * G * 8 >= (size_t)p.W * G * 16) {
    p.WP = p.R;
  } else {
    p.WP = o; o = al(o + 16 * (size_t)p.W * G);
  }
  p.total = o;
  return p;
}

}  // namespace wide

// NM: run_precoding's NMSE stop (solvers.py:583-603) -- the system's ceil(K / 32) CTAs form one thread-block
// cluster, evaluate err = ||F_ref - M / ||M|| || / ||F_ref|| after every outer iteration from the register-resident
// iterate (two fixed-order fp64 reductions exchanged over DSMEM) and leave together at the first err < eps, at
// all-done or at the cap T
template <int SCH, bool NM>
__global__ void __launch_bounds__(512, 1) kz_wide_kernel(const __grid_constant__ LsArgs p) {
  using namespace wide;
  using T = float2;
  constexpr bool PER_LANE_ROW = SCH == KZ_URK || SCH == KZ_SWOR_ERK;
  constexpr bool AGG = SCH == KZ_AHK || SCH == KZ_VR_OAHK;
  // measured per scheme (same-box A/B, tools/ab3.sh): half pieces in their own list segments, and the aggregation
  // weights formed by the whole CTA (PAR_W) instead of one half-warp per rhs
  constexpr bool HALF = (KZ_WIDE_HALF_MASK >> SCH) & 1;
  constexpr bool PAR_W = AGG && ((KZ_WIDE_PARW_MASK >> SCH) & 1);

  extern __shared__ __align__(16) unsigned char sm[];
  const int K = p.P.n_users, Nt = p.P.n_antennas;
  const int ngroups = (K + G - 1) / G;
  const int b = blockIdx.x / ngroups, grp = blockIdx.x % ngroups, g0 = grp * G;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int nthr = blockDim.x;
  const Plan pl = plan(K, Nt, p.S, p.hcap);
  const int W = pl.W, SL = pl.SL, KW = (K + 31) / 32;

  int* rowS = (int*)(sm + pl.rowS);
  int* rowL = (int*)(sm + pl.rowL);
  int* c0 = (int*)(sm + pl.c0);
  int* c1 = (int*)(sm + pl.c1);
  int* hoff = (int*)(sm + pl.hoff);  // element index of antenna CH*c0 of row i
  float* en = (float*)(sm + pl.en);
  float* inv_en = (float*)(sm + pl.inv_en);  // 1 / e_i (aggregation weights phi = r / e)
  long long* cost = (long long*)(sm + pl.cost);
  uint32_t* cmask = (uint32_t*)(sm + pl.cmask);
  int* lptr = (int*)(sm + pl.lptr);
  int2* lst = (int2*)(sm + pl.lst);  // (h element offset of this chunk, P offset of this (row, slot))
  T* Hs = (T*)(sm + pl.H);
  T* Ps = (T*)(sm + pl.P);
  T* Qs = (T*)(sm + pl.Q);
  T* Rs = (T*)(sm + pl.R);
  int* sel = (int*)(sm + pl.sel);
  T* gam = (T*)(sm + pl.gam);
  int* donev = (int*)(sm + pl.done);
  int* itv = (int*)(sm + pl.iters);
  long long* flv = (long long*)(sm + pl.flops);
  int* prevv = (int*)(sm + pl.prev);
  uint32_t* poolv = (uint32_t*)(sm + pl.pool);
  int* poolcnt = (int*)(sm + pl.poolcnt);
  uint8_t* inset = (uint8_t*)(sm + pl.inset);
  int* optr = (int*)(sm + pl.optr);
  int2* olst = (int2*)(sm + pl.olst);
  int* nptr = (int*)(sm + pl.nptr);
  int2* nlst = (int2*)(sm + pl.nlst);
  T* Phi = (T*)(sm + pl.Phi);
  float* Dp = (float*)(sm + pl.Dp);
  T* numv = (T*)(sm + pl.num);
  float* spv = (float*)(sm + pl.sp);
  int* nzv = (int*)(sm + pl.nz);
  int* noopv = (int*)(sm + pl.noop);
  uint32_t* misc = (uint32_t*)(sm + pl.misc);

  const float regf = (float)p.P.reg[b];
  const T* heff = (const T*)p.P.heff;
  KZ_TSTART

  // ------------------------------------------------------------------ setup
  for (int i = tid; i < K; i += nthr) {
    size_t r = (size_t)b * K + i;
    int sg = p.P.row_seg_ptr[r];
    int s = p.P.seg_start[sg], L = p.P.seg_len[sg];
    rowS[i] = s;
    rowL[i] = L;
    c0[i] = s / CH;
    c1[i] = (s + L - 1) / CH;
    en[i] = (float)p.P.row_energy[r];
    inv_en[i] = (float)(1.0 / p.P.row_energy[r]);
  }
  __syncthreads();
  // padded row offsets (prefix over rows) by warp 0
  if (w == 0) {
    int carry = 0;
    for (int base = 0; base < K; base += 32) {
      int i = base + lane;
      // each row is followed by one spare 16-byte unit, so row i starts at bank group i mod 8 (16-byte units mod 128
      // bytes; the chunk-padded rows alone are multiples of 256 bytes): the eight rows a quarter-warp's LDS.128
      // gathers in the projection (one row per rhs lane) then spread over all eight groups instead of sharing one
      int v = i < K ? (c1[i] - c0[i] + 1) * CH + HSKEW : 0;
      int sc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int t2 = __shfl_up_sync(FULL, sc, o);
        if (lane >= o) sc += t2;
      }
      if (i < K) hoff[i] = carry + sc - v;
      carry += __shfl_sync(FULL, sc, 31);
    }
  }
  // partition flags: 1 = orthogonal group O, 2 = non-orthogonal N (vrgraph.py:84-114)
  for (int i = tid; i < K; i += nthr) inset[i] = 0;
  __syncthreads();
  if (AGG && p.P.orth_ptr) {
    for (int q = p.P.orth_ptr[b] + tid; q < p.P.orth_ptr[b + 1]; q += nthr) inset[p.P.orth_idx[q]] = 1;
    for (int q = p.P.non_ptr[b] + tid; q < p.P.non_ptr[b + 1]; q += nthr) inset[p.P.non_idx[q]] = 2;
  }
  __syncthreads();
  // per-chunk row lists (all rows / O / N): warp w compacts with ballots, in three segments of ascending rows --
  // the pieces whose support covers both 16-antenna halves of the chunk, then those touching only the first half,
  // then only the second half (spl[2 w], spl[2 w + 1]: segment starts): a half piece needs half the loads and FMAs
  // (the other half of the chunk is zero padding), and a row of L = 128 at a random start has one of its 4-5 pieces
  // in that case.  entry = (h element offset of this chunk | row << 20,
  //                          P offset of (row, slot) | (row & 15) | half-chunk mask << 28)
  auto build_list = [&](int* ptr, int* spl, int2* out, int which) {
    auto half_mask = [&](int i) {  // which 16-antenna halves of this chunk the row's support touches
      const int lo = rowS[i] - w * CH, hi = rowS[i] + rowL[i] - w * CH;
      return (lo < 16 && hi > 0 ? 1 : 0) | (lo < 32 && hi > 16 ? 2 : 0);
    };
    int n = 0, nf = 0, nl = 0;
    for (int base = 0; base < K; base += 32) {
      int i = base + lane;
      bool ov = i < K && c0[i] <= w && w <= c1[i] && (which == 0 || inset[i] == which);
      const int hm = ov ? half_mask(i) : 0;
      n += __popc(__ballot_sync(FULL, ov));
      nf += __popc(__ballot_sync(FULL, ov && (hm == 3 || !HALF)));
      nl += __popc(__ballot_sync(FULL, ov && hm == 1 && HALF));
    }
    if (lane == 0) ptr[w + 1] = n;
    __syncthreads();
    if (tid == 0) {
      ptr[0] = 0;
      for (int ww = 0; ww < W; ++ww) ptr[ww + 1] += ptr[ww];
    }
    __syncthreads();
    int q[3] = {ptr[w], ptr[w] + nf, ptr[w] + nf + nl};
    if (lane == 0) {
      spl[2 * w] = q[1];
      spl[2 * w + 1] = q[2];
    }
    for (int base = 0; base < K; base += 32) {
      int i = base + lane;
      bool ov = i < K && c0[i] <= w && w <= c1[i] && (which == 0 || inset[i] == which);
      const int hm = ov ? half_mask(i) : 0;
      const int seg = (hm == 3 || !HALF) ? 0 : (hm == 1 ? 1 : 2);
#pragma unroll
      for (int sg = 0; sg < 3; ++sg) {
        const unsigned bal = __ballot_sync(FULL, ov && seg == sg);
        if (ov && seg == sg) {
          const int slot = w - c0[i];
          out[q[sg] + __popc(bal & ((1u << lane) - 1))] =
              make_int2((hoff[i] + slot * CH) | (i << 20), (i * SL + slot) * G | (i & 15) | (hm << 28));
        }
        q[sg] += __popc(bal);
      }
    }
  };
  __syncthreads();  // hoff ready
  int* lspl = (int*)(sm + pl.lspl);
  int* ospl = (int*)(sm + pl.ospl);
  int* nspl = (int*)(sm + pl.nspl);
  KZ_CHECK(tid >= K || hoff[tid] + (c1[tid] - c0[tid] + 1) * CH <= pl.hcap, "wide: row layout inside H");
  if (SCH != KZ_VR_OAHK) build_list(lptr, lspl, lst, 0);
  if (SCH == KZ_VR_OAHK) {
    build_list(optr, ospl, olst, 1);
    build_list(nptr, nspl, nlst, 2);
  }
  // TMEM: 4 warps per 32-lane subpartition x 64 columns (2 rhs x 16 complex antennas) each
  if constexpr (AGG) {
    if (w == 0) tmem::alloc(misc, 256);
    tmem::fence_before();
  }
  // rows -> shared memory, zero padded to whole chunks: one bulk copy per row whose packed offset has its first
  // antenna's parity (kz_tma.cuh; warp per row, lane 0 issues), 8-byte asynchronous copies for the others, then
  // the first / last piece's antennas outside the support are zeroed
  {
    uint64_t* mbar = (uint64_t*)(sm + pl.mbar);
    const bool bulk = p.bulk != 0;
    if (bulk && tid == 0) tma::mbar_init(mbar, 1);
    __syncthreads();
    for (int i = w; i < K; i += W) {
      const int s = rowS[i], L = rowL[i], np = c1[i] - c0[i] + 1;
      const long long rvo = p.P.row_val_ptr[(size_t)b * K + i];
      int done = 0;
      if (lane == 0 && bulk)
        done = tma::stage_run_bulk(Hs + hoff[i], heff, rvo, s, L, c0[i] * CH, (c1[i] + 1) * CH, p.P.val_lo,
                                   p.P.val_hi, mbar);
      if (!__shfl_sync(FULL, done, 0))
        for (int pc = 0; pc < np; ++pc) {
          const int ant = (c0[i] + pc) * CH + lane;
          const bool in = ant >= s && ant < s + L;
          cp_async8(Hs + hoff[i] + pc * CH + lane, heff + rvo + (in ? ant - s : 0), in);
        }
    }
    if (bulk) {
      __syncthreads();
      if (tid == 0) tma::mbar_arrive(mbar);
    }
    cp_async_wait_all();
    if (bulk) {
      tma::mbar_wait(mbar, 0);
      for (int i = w; i < K; i += W) {
        const int np = c1[i] - c0[i];
        for (int pc = 0; pc <= np; pc += max(1, np)) {
          const int ant = (c0[i] + pc) * CH + lane;
          if (ant < rowS[i] || ant >= rowS[i] + rowL[i]) Hs[hoff[i] + pc * CH + lane] = make_float2(0.f, 0.f);
        }
      }
    }
  }
  // vr-oahk: the O rows in ascending order (in cmask, which only vr-ogrk uses) and their count (misc[1]): the
  // block step hands row k of the list to warp k, the other warps go straight to the barrier
  int* orow = (int*)cmask;
  if constexpr (SCH == KZ_VR_OAHK) {
    if (w == 0) {
      int n = 0;
      for (int base = 0; base < K; base += 32) {
        const int i = base + lane;
        const bool o = i < K && inset[i] == 1;
        const unsigned bal = __ballot_sync(FULL, o);
        if (o) orow[n + __popc(bal & ((1u << lane) - 1))] = i;
        n += __popc(bal);
      }
      if (lane == 0) misc[1] = (uint32_t)n;
    }
  }
  if constexpr (SCH == KZ_VR_OGRK) {
    for (int i = tid; i < K; i += nthr) {
      size_t r = (size_t)b * K + i;
      long long cst = 0;
      for (int q = 0; q < KW; ++q) cmask[i * KW + q] = 0;
      for (int q = p.P.coupled_ptr[r]; q < p.P.coupled_ptr[r + 1]; ++q) {
        int j = p.P.coupled_idx[q];
        cmask[i * KW + (j >> 5)] |= 1u << (j & 31);
        cst += 8LL * rowL[j] + 4;
      }
      cost[i] = cst;
    }
  }
  for (int e = tid; e < K * G; e += nthr) {
    int i = e / G, gg = e % G;
    Qs[xs(i, gg)] = make_float2(0.f, 0.f);
    Rs[xs(i, gg)] = make_float2(i == g0 + gg ? 1.f : 0.f, 0.f);
  }
  for (int gg = tid; gg < G; gg += nthr) {
    donev[gg] = (g0 + gg < K) ? 0 : 1;
    itv[gg] = 0;
    flv[gg] = 0;
    prevv[gg] = -1;
    poolcnt[gg] = 0;
    sel[gg] = -1;
    noopv[gg] = 0;
    nzv[gg] = 0;
  }
  __syncthreads();
  KZ_PHASE();
  KZ_CHECK(SCH == KZ_VR_OAHK || lptr[W] <= K * SL, "wide: piece list capacity");
  KZ_CHECK(SCH != KZ_VR_OAHK || (optr[W] <= K * SL && nptr[W] <= K * SL), "wide: O / N piece list capacity");
  KZ_CHECK(!AGG || W <= 16, "wide: TMEM columns (4 warps x 64 per lane quarter)");
  KZ_CHECK(!AGG || pl.WP != pl.R || (size_t)W * G * 16 <= (size_t)K * G * 8, "wide: weight partials inside R");
  uint32_t my_tmem = 0;
  if constexpr (AGG) {
    tmem::fence_after();
    my_tmem = misc[0] + ((uint32_t)(32 * (w & 3)) << 16) + 64u * (uint32_t)(w >> 2);
  }
  long long costO = 0, costN = 0;
  int nN = 0;
  for (int i = 0; i < K; ++i) {
    if (inset[i] == 1) costO += 8LL * rowL[i] + 4;
    if (inset[i] == 2) { costN += 8LL * rowL[i]; ++nN; }
  }
  const int unionN = (AGG && p.P.non_union_size) ? p.P.non_union_size[b] : 0;

  // NMSE-stopped runs: ||F_ref|| of the whole system (every CTA of the cluster forms the same fixed-order sum)
  const NmxSlots nms = nmx_slots(sm + pl.nmx);
  double* red = (double*)(sm + pl.red);
  const bool need_err = NM && (p.eps > 0.0 || p.O.nmse_trace);
  const double* fref = need_err ? p.f_ref + (size_t)b * Nt * K * 2 : nullptr;
  double fref_norm = 0.0;
  if constexpr (NM) {
    if (need_err) {
      double s2 = 0.0;
      const double2* f2 = reinterpret_cast<const double2*>(fref);
      for (int e = tid; e < Nt * K; e += nthr) {
        const double2 f = __ldg(f2 + e);
        s2 = fma(f.x, f.x, fma(f.y, f.y, s2));
      }
      fref_norm = sqrt(cta_sum_d(s2, red, w, lane, W));
    }
    cluster_barrier();  // every CTA of the system is resident before the first DSMEM store
  }
  bool conv = false;

  constexpr int E = 16;  // antennas per thread per chunk
  const int a = lane >> 4, g = lane & 15;
  T m0[E], m1[E];  // rhs g and g + 16
#pragma unroll
  for (int k = 0; k < E; ++k) m0[k] = m1[k] = make_float2(0.f, 0.f);
  const float4* H4 = reinterpret_cast<const float4*>(Hs);
  // antenna of element k of this thread within the chunk: 4*(k/2) + 2a + (k&1)

  // conj(h) . m for both rhs over the chunk; returns this lane's rhs partial after
  // the a-lane exchange (lane a keeps rhs g + 16a)
  // j range [J0, J1) of the thread's 8 float4 pairs: <0, 8> = the whole chunk, <0, 4> / <4, 8> = the first /
  // second 16 antennas (a half piece: the rest of the chunk is zero padding, skipping it is exact)
  auto dot_part = [&](auto jr, int h0) -> T {
    constexpr int J0 = decltype(jr)::lo, J1 = decltype(jr)::hi;
    KZ_CHECK(h0 >= 0 && (h0 & 1) == 0 && h0 + CH <= pl.hcap, "wide: refresh piece inside H");
    const float4* hp = H4 + ((h0 + 2 * a) >> 1);
    float x0 = 0.f, y0 = 0.f, x1 = 0.f, y1 = 0.f, u0 = 0.f, v0 = 0.f, u1 = 0.f, v1 = 0.f;
    {
#pragma unroll
      for (int j = J0; j < J1; ++j) {
        float4 h = hp[2 * j];
        const int k = 2 * j;
        x0 = fmaf(h.x, m0[k].x, x0); x0 = fmaf(h.y, m0[k].y, x0);
        y0 = fmaf(h.x, m0[k].y, y0); y0 = fmaf(-h.y, m0[k].x, y0);
        x1 = fmaf(h.z, m0[k + 1].x, x1); x1 = fmaf(h.w, m0[k + 1].y, x1);
        y1 = fmaf(h.z, m0[k + 1].y, y1); y1 = fmaf(-h.w, m0[k + 1].x, y1);
        u0 = fmaf(h.x, m1[k].x, u0); u0 = fmaf(h.y, m1[k].y, u0);
        v0 = fmaf(h.x, m1[k].y, v0); v0 = fmaf(-h.y, m1[k].x, v0);
        u1 = fmaf(h.z, m1[k + 1].x, u1); u1 = fmaf(h.w, m1[k + 1].y, u1);
        v1 = fmaf(h.z, m1[k + 1].y, v1); v1 = fmaf(-h.w, m1[k + 1].x, v1);
      }
    }
    const float px = x0 + x1, py = y0 + y1, qx = u0 + u1, qy = v0 + v1;
    // lane a keeps rhs g + 16a: send the other rhs' partial to the partner lane
    const float sx = a ? px : qx, sy = a ? py : qy;
    const float rx = __shfl_xor_sync(FULL, sx, 16), ry = __shfl_xor_sync(FULL, sy, 16);
    return a ? make_float2(qx + rx, qy + ry) : make_float2(px + rx, py + ry);
  };
  // P element of list entry e for this lane's rhs
  auto pslot = [&](int ey) {
    const int o = (ey & 0x0FFFFFE0) + ((g + 16 * a) ^ (ey & 15));
    KZ_CHECK(o >= 0 && o < K * SL * G, "wide: P slot index");
    return o;
  };
  // partials of the list entries [q, q1) -> P, NF pieces in flight (1, 2 or 4)
  auto refresh_seg = [&](auto jr, auto nf, const int2* L, int q, const int q1) {
    constexpr int NF = decltype(nf)::value;
    if constexpr (NF >= 4) {
      for (; q + 3 < q1; q += 4) {
        const int2 e0 = L[q], e1 = L[q + 1], e2 = L[q + 2], e3 = L[q + 3];
        const T v0 = dot_part(jr, e0.x & 0xFFFFF);
        const T v1 = dot_part(jr, e1.x & 0xFFFFF);
        const T v2 = dot_part(jr, e2.x & 0xFFFFF);
        const T v3 = dot_part(jr, e3.x & 0xFFFFF);
        Ps[pslot(e0.y)] = v0;
        Ps[pslot(e1.y)] = v1;
        Ps[pslot(e2.y)] = v2;
        Ps[pslot(e3.y)] = v3;
      }
    }
    for (; q + 1 < q1; q += 2) {
      const int2 e0 = L[q], e1 = L[q + 1];
      const T v0 = dot_part(jr, e0.x & 0xFFFFF);
      const T v1 = dot_part(jr, e1.x & 0xFFFFF);
      Ps[pslot(e0.y)] = v0;
      Ps[pslot(e1.y)] = v1;
    }
    if (q < q1) {
      const int2 e0 = L[q];
      Ps[pslot(e0.y)] = dot_part(jr, e0.x & 0xFFFFF);
    }
  };
  // refresh partials of warp w's pieces of a list: whole-chunk pieces (four in flight; vr-oahk two: its larger
  // live state would spill), then the first-half and second-half pieces (two in flight)
  auto refresh_list = [&](const int* ptr, const int* spl, const int2* L) {
    using NF = std::integral_constant<int, SCH == KZ_VR_OAHK ? 2 : KZ_WIDE_NF>;
    refresh_seg(JRange<0, 8>{}, NF{}, L, ptr[w], spl[2 * w]);
    if constexpr (HALF) {
      refresh_seg(JRange<0, 4>{}, std::integral_constant<int, 2>{}, L, spl[2 * w], spl[2 * w + 1]);
      refresh_seg(JRange<4, 8>{}, std::integral_constant<int, 2>{}, L, spl[2 * w + 1], ptr[w + 1]);
    }
  };
  // bt: every slot load issued at once (predicated), then the sums in slot order -- for callers with registers to
  // spare (the greedy selection; the aggregation weights, formed while the iterate is parked in TMEM)
  auto resid_q = [&](auto bt, int i, int gg, const T q) -> T {  // from the slot partials, fixed order; q = q_i
    KZ_CHECK(i >= 0 && i < K && gg >= 0 && gg < G && c1[i] - c0[i] < SL, "wide: residual row / slots");
    const T* pp = Ps + (size_t)i * SL * G + (gg ^ (i & 15));
    float dx = 0.f, dy = 0.f;
    const int ns = c1[i] - c0[i];
    if (decltype(bt)::value && SL <= 8) {
      T v[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) v[s] = s <= ns ? pp[(size_t)s * G] : make_float2(0.f, 0.f);
#pragma unroll
      for (int s = 0; s < 8; ++s)
        if (s <= ns) {
          dx += v[s].x;
          dy += v[s].y;
        }
    } else {
      for (int s = 0; s <= ns; ++s) {
        T v = pp[(size_t)s * G];
        dx += v.x;
        dy += v.y;
      }
    }
    const int c = g0 + gg;
    if (SCH == KZ_GK || SCH == KZ_GRK || SCH == KZ_AHK) {  // dense form (solvers.py:149-153)
      T r = make_float2(-dx - q.x * regf, -dy - q.y * regf);
      if (i == c) r.x += 1.f;
      return r;
    }
    float tg = i == c ? 1.f : 0.f;  // VR form (solvers.py:166)
    return make_float2((tg - dx) - q.x * regf, (0.f - dy) - q.y * regf);
  };
  auto resid_b = [&](auto bt, int i, int gg) -> T { return resid_q(bt, i, gg, Qs[xs(i, gg)]); };
  auto resid = [&](int i, int gg) -> T { return resid_b(std::bool_constant<SCH != KZ_VR_OAHK>{}, i, gg); };
  auto draw_u = [&](int gg) -> double {
    int c = g0 + gg, d = itv[gg];
    if (p.R.kind == KZ_RNG_PHILOX) return philox_uniform(p.R.seed, (uint32_t)(b + p.R.system_base), (uint32_t)c, (uint64_t)d);
    return p.R.uniforms[((size_t)b * K + c) * p.R.stream_len + d];
  };
  auto take_step = [&](int gg, int i, T r, long long f) {
    const float e = en[i];
    T gm = make_float2(r.x / e, r.y / e);
    T q = Qs[xs(i, gg)];
    Qs[xs(i, gg)] = make_float2(q.x + gm.x, q.y + gm.y);
    Rs[xs(i, gg)] = make_float2(0.f, 0.f);
    gam[gg] = gm;
    sel[gg] = i;
    const int it = itv[gg];
    if (p.O.rows && it < p.O.rows_cap) p.O.rows[((size_t)b * K + g0 + gg) * p.O.rows_cap + it] = i;
    itv[gg] = it + 1;
    flv[gg] += f;
  };
  // m_r += gm h_i on this thread's antennas of the chunk (rows zero padded => whole chunk)
  auto project = [&](T (&mr)[E], int i, T gm) {
    if (i < 0 || w < c0[i] || w > c1[i]) return;
    KZ_CHECK(i < K && hoff[i] + (w - c0[i] + 1) * CH <= pl.hcap, "wide: projected piece inside H");
    const float4* hp = H4 + ((hoff[i] + (w - c0[i]) * CH + 2 * a) >> 1);
#pragma unroll
    for (int j = 0; j < E / 2; ++j) {
      float4 h = hp[2 * j];
      const int k = 2 * j;
      mr[k].x = fmaf(gm.x, h.x, mr[k].x); mr[k].x = fmaf(-gm.y, h.y, mr[k].x);
      mr[k].y = fmaf(gm.x, h.y, mr[k].y); mr[k].y = fmaf(gm.y, h.x, mr[k].y);
      mr[k + 1].x = fmaf(gm.x, h.z, mr[k + 1].x); mr[k + 1].x = fmaf(-gm.y, h.w, mr[k + 1].x);
      mr[k + 1].y = fmaf(gm.x, h.w, mr[k + 1].y); mr[k + 1].y = fmaf(gm.y, h.z, mr[k + 1].y);
    }
  };

  const long long dense_refresh = 6LL * K * Nt + 2LL * K * (Nt + 1) + 2LL * K;
  const long long dense_rk = 2 + 8LL * Nt + 2;
  int t;
  for (t = 1; t <= p.T; ++t) {
    KZ_ITER();
    if constexpr (SCH == KZ_GK || SCH == KZ_GRK || SCH == KZ_VR_OGRK) {
      refresh_list(lptr, lspl, lst);  // every row overlapping this chunk
      KZ_WSTAMP();
      __syncthreads();
      KZ_PHASE();
      // finalise + select: each half-warp serves one rhs (lanes over rows, 16-lane scans)
      {
        const int hf = lane >> 4, hl = lane & 15;
        const unsigned hmask = 0xFFFFu << (16 * hf);
        for (int pair = w; pair < G / 2; pair += W) {
          const int gg = pair + hf * (G / 2);
          const bool act = g0 + gg < K && !donev[gg];
          double u = 0.0;
          if (SCH != KZ_GK && act) u = draw_u(gg);  // independent of the residuals: issue early
          float wsum = 0.f;
          if (act)
#pragma unroll 4
            for (int i = hl; i < K; i += 16) {
              T r;
              if constexpr (SCH == KZ_VR_OGRK) {
                // only the rows coupled to the previous pick take their new residual (solvers.py:398-406); the
                // slot sums of all four rows of the lane are formed without branches (loads in flight together)
                // and the uncoupled rows keep the stored value
                const int pr = prevv[gg];
                const bool upd = pr >= 0 && ((cmask[pr * KW + (i >> 5)] >> (i & 31)) & 1u);
                const T rn = resid(i, gg), ro = Rs[xs(i, gg)];
                r = upd ? rn : ro;
                if (upd) Rs[xs(i, gg)] = r;
              } else {
                r = resid(i, gg);
                Rs[xs(i, gg)] = r;
              }
              wsum += r.x * r.x + r.y * r.y;
            }
          __syncwarp();
          KZ_PHASE();  // [timing] residuals of this rhs' rows
          int isel = -1;
          long long f;
          if constexpr (SCH == KZ_GK) {
            float best = -1.f;
            int bi = 0x7fffffff;
            bool any = false;
            if (act)
              for (int i = hl; i < K; i += 16) {
                T r = Rs[xs(i, gg)];
                float sc = (r.x * r.x + r.y * r.y) / en[i];
                if (sc != 0.f) any = true;
                if (sc > best) { best = sc; bi = i; }
              }
            for (int o = 8; o > 0; o >>= 1) {
              float ob = __shfl_xor_sync(FULL, best, o);
              int oi = __shfl_xor_sync(FULL, bi, o);
              if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
            }
            isel = (__ballot_sync(FULL, any) & hmask) ? bi : -1;
            f = dense_refresh + 4LL * K;
          } else {
            float tot = wsum;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) tot += __shfl_xor_sync(FULL, tot, o);
            f = (SCH == KZ_GRK ? dense_refresh : (prevv[gg] >= 0 ? cost[prevv[gg]] : 0)) + 4LL * K + 2;
            const float tau = (float)u * tot;
            float carry = 0.f;
            int lastnz = -1;
            bool found = !(tot > 0.f);  // tot == 0: None, no draw is consumed (solvers.py:235-236)
            // rows in blocks of 64, lane hl owning 4 consecutive rows: one 16-lane scan per block
            for (int base = 0; base < K; base += 64) {
              if (__all_sync(FULL, found)) break;
              float wt[4], ls = 0.f;
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                const int i = base + 4 * hl + t;
                float v = 0.f;
                if (act && i < K) {
                  const T r = Rs[xs(i, gg)];
                  v = r.x * r.x + r.y * r.y;
                }
                wt[t] = v;
                ls += v;
              }
              float sc = ls;
#pragma unroll
              for (int o = 1; o < 16; o <<= 1) {
                const float t2 = __shfl_up_sync(FULL, sc, o, 16);
                if (hl >= o) sc += t2;
              }
              float run = carry + sc - ls;  // weight before this lane's first row
              int lt = -1, lnz = -1;
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                run += wt[t];
                if (lt < 0 && wt[t] > 0.f && run > tau) lt = t;
                if (wt[t] > 0.f) lnz = t;
              }
              const unsigned bal = (__ballot_sync(FULL, !found && lt >= 0) & hmask) >> (16 * hf);
              const unsigned nzb = (__ballot_sync(FULL, lnz >= 0) & hmask) >> (16 * hf);
              const int srcl = bal ? __ffs(bal) - 1 : 0, srcn = nzb ? 31 - __clz(nzb) : 0;
              const int lt_s = __shfl_sync(FULL, lt, 16 * hf + srcl);
              const int lnz_s = __shfl_sync(FULL, lnz, 16 * hf + srcn);
              if (!found && bal) {
                isel = base + 4 * srcl + lt_s;
                found = true;
              }
              if (nzb) lastnz = base + 4 * srcn + lnz_s;
              carry += __shfl_sync(FULL, sc, 16 * hf + 15);
            }
            if (tot > 0.f && isel < 0) isel = lastnz;
          }
          KZ_PHASE();  // [timing] row pick
          if (hl == 0 && act) {
            if (isel < 0) {
              donev[gg] = 1;
              sel[gg] = -1;
              flv[gg] += f;
            } else {
              long long fr = SCH == KZ_VR_OGRK ? 2 + 8LL * rowL[isel] + 2 : dense_rk;
              take_step(gg, isel, Rs[xs(isel, gg)], f + fr);
              if constexpr (SCH == KZ_VR_OGRK) prevv[gg] = isel;
            }
          } else if (hl == 0) {
            sel[gg] = -1;
          }
          __syncwarp();
        }
      }
      __syncthreads();
      KZ_PHASE();
      project(m0, sel[g], gam[g]);
      project(m1, sel[g + 16], gam[g + 16]);
    } else if constexpr (PER_LANE_ROW) {
      // row draw per rhs (host index stream / Philox), one thread per rhs
      if (tid < G) {
        const int gg = tid;
        int i = -1;
        if (g0 + gg < K && !donev[gg]) {
          const int c = g0 + gg, d = itv[gg];
          long long f = SCH == KZ_SWOR_ERK ? (K - d % K) + 2 : 0;
          if (p.R.kind == KZ_RNG_HOST_INDEX) {
            i = p.R.indices[((size_t)b * K + c) * p.R.stream_len + d];
          } else if (SCH == KZ_URK) {
            i = (int)(draw_u(gg) * K);
            i = i >= K ? K - 1 : i;
          } else {
            uint32_t* pbm = poolv + gg * KW;
            if (poolcnt[gg] == 0) {
              for (int q = 0; q < KW; ++q) pbm[q] = 0;
              for (int j = 0; j < K; ++j) pbm[j >> 5] |= 1u << (j & 31);
              poolcnt[gg] = K;
            }
            double tot = 0.0;
            for (int j = 0; j < K; ++j)
              if ((pbm[j >> 5] >> (j & 31)) & 1u) tot += p.P.row_energy[(size_t)b * K + j];
            double u = draw_u(gg) * tot, acc = 0.0;
            int last = -1;
            for (int j = 0; j < K; ++j) {
              if (!((pbm[j >> 5] >> (j & 31)) & 1u)) continue;
              last = j;
              acc += p.P.row_energy[(size_t)b * K + j];
              if (acc > u) { i = j; break; }
            }
            if (i < 0) i = last;
            pbm[i >> 5] &= ~(1u << (i & 31));
            poolcnt[gg] -= 1;
          }
          flv[gg] += f;
        }
        sel[gg] = i;
      }
      __syncthreads();
      KZ_PHASE();
      {  // partials of the lanes' own rows on this chunk (gathered loads), rhs g then g + 16
        auto own_row = [&](const T (&mr)[E], int r) {
          const int i = sel[g + 16 * r];
          const bool ov = i >= 0 && w >= c0[i] && w <= c1[i];
          float px = 0.f, py = 0.f;
          if (ov) {
            const float4* hp = H4 + ((hoff[i] + (w - c0[i]) * CH + 2 * a) >> 1);
#pragma unroll
            for (int j = 0; j < E / 2; ++j) {
              float4 h = hp[2 * j];
              const int k = 2 * j;
              px = fmaf(h.x, mr[k].x, px); px = fmaf(h.y, mr[k].y, px);
              py = fmaf(h.x, mr[k].y, py); py = fmaf(-h.y, mr[k].x, py);
              px = fmaf(h.z, mr[k + 1].x, px); px = fmaf(h.w, mr[k + 1].y, px);
              py = fmaf(h.z, mr[k + 1].y, py); py = fmaf(-h.w, mr[k + 1].x, py);
            }
          }
          px += __shfl_xor_sync(FULL, px, 16);
          py += __shfl_xor_sync(FULL, py, 16);
          if (ov && a == r) Ps[(size_t)(i * SL + (w - c0[i])) * G + ((g + 16 * r) ^ (i & 15))] = make_float2(px, py);
        };
        own_row(m0, 0);
        own_row(m1, 1);
      }
      __syncthreads();
      KZ_PHASE();
      if (tid < G) {
        const int i = sel[tid];
        if (i >= 0) take_step(tid, i, resid(i, tid), 2 * (8LL * Nt + 4));
      }
      __syncthreads();
      KZ_PHASE();
      project(m0, sel[g], gam[g]);
      project(m1, sel[g + 16], gam[g + 16]);
      __syncthreads();  // sel/gam are rewritten by the next draw
    } else {  // AHK / VR-OAHK (solvers.py:407-421)
      // residuals -> weights phi = r/e, num = vdot(phi, r), ||phi||^2 (solvers.py:248-254, 274) with the whole
      // CTA: thread (w, lane) takes rows w, w + W, ... of rhs lane and leaves its partial sums in WP[w][lane];
      // warp 0 reduces them per rhs in warp order (reduce_weights) once the partials are visible
      float2* WPn = (float2*)(sm + pl.WP);
      float* WPs = (float*)(sm + pl.WP + 8 * (size_t)W * G);
      int* WPz = (int*)(sm + pl.WP + 12 * (size_t)W * G);
      auto weights = [&](int which) {
        const int gg = lane;
        float nx = 0.f, ny = 0.f, sp = 0.f;
        bool nz = false;
        // the previous aggregated step's q += gamma phi on these rows is applied here, where q_i is loaded
        // anyway (sel / gam: that step's flag and length per rhs; the old phi is still in Phi)
        const bool pend = sel[gg] > 0;
        const T pg = gam[gg];
        if (g0 + gg < K && !donev[gg])
#pragma unroll 4
          for (int i = w; i < K; i += W) {
            if (which && inset[i] != which) continue;
            T q = Qs[xs(i, gg)];
            if (pend) {
              q = cfma(pg, Phi[xs(i, gg)], q);
              Qs[xs(i, gg)] = q;
            }
            const T r = resid_q(std::true_type{}, i, gg, q);
            const float ie = inv_en[i];
            const T ph = make_float2(r.x * ie, r.y * ie);
            Phi[xs(i, gg)] = ph;
            nz |= (ph.x != 0.f || ph.y != 0.f);
            nx = fmaf(ph.x, r.x, nx); nx = fmaf(ph.y, r.y, nx);
            ny = fmaf(ph.x, r.y, ny); ny = fmaf(-ph.y, r.x, ny);
            sp = fmaf(ph.x, ph.x, sp); sp = fmaf(ph.y, ph.y, sp);
          }
        WPn[w * G + gg] = make_float2(nx, ny);
        WPs[w * G + gg] = sp;
        WPz[w * G + gg] = nz ? 1 : 0;
      };
      auto reduce_weights = [&](int nrows) {  // warp 0, lane = rhs slot
        if (w != 0) return;
        const int gg = lane;
        float nx = 0.f, ny = 0.f, sp = 0.f;
        int anz = 0;
        for (int ww = 0; ww < W; ++ww) {
          const float2 n2 = WPn[ww * G + gg];
          nx += n2.x;
          ny += n2.y;
          sp += WPs[ww * G + gg];
          anz |= WPz[ww * G + gg];
        }
        if (g0 + gg < K && !donev[gg]) {
          numv[gg] = make_float2(nx, ny);
          spv[gg] = sp;
          nzv[gg] = (anz && nrows > 0) ? 1 : 0;
          flv[gg] += 2LL * nrows;
        } else {
          nzv[gg] = 0;
        }
      };
      // the same with one half-warp per rhs (lanes over rows, shuffle reductions): the AHK form
      auto weights_rhs = [&](int which, int nrows) {
        const int hf = lane >> 4, hl = lane & 15;  // one half-warp per rhs, lanes over rows
        const unsigned hmask = 0xFFFFu << (16 * hf);
        for (int pair = w; pair < G / 2; pair += W) {
          const int gg = pair + hf * (G / 2);
          const bool act = g0 + gg < K && !donev[gg];
          float nx = 0.f, ny = 0.f, sp = 0.f;
          bool nz = false;
          const bool pend = sel[gg] > 0;  // the previous step's q += gamma phi, applied where q_i is loaded
          const T pg = gam[gg];
          if (act)
#pragma unroll 4
            for (int i = hl; i < K; i += 16) {
              if (which && inset[i] != which) continue;
              T q = Qs[xs(i, gg)];
              if (pend) {
                q = cfma(pg, Phi[xs(i, gg)], q);
                Qs[xs(i, gg)] = q;
              }
              const T r = resid_q(std::true_type{}, i, gg, q);
              const float ie = inv_en[i];
              const T ph = make_float2(r.x * ie, r.y * ie);
              Phi[xs(i, gg)] = ph;
              nz |= (ph.x != 0.f || ph.y != 0.f);
              nx = fmaf(ph.x, r.x, nx); nx = fmaf(ph.y, r.y, nx);
              ny = fmaf(ph.x, r.y, ny); ny = fmaf(-ph.y, r.x, ny);
              sp = fmaf(ph.x, ph.x, sp); sp = fmaf(ph.y, ph.y, sp);
            }
#pragma unroll
          for (int o = 8; o > 0; o >>= 1) {
            nx += __shfl_xor_sync(FULL, nx, o);
            ny += __shfl_xor_sync(FULL, ny, o);
            sp += __shfl_xor_sync(FULL, sp, o);
          }
          const bool anz = (__ballot_sync(FULL, nz) & hmask) != 0;
          if (hl == 0) {
            if (act) {
              numv[gg] = make_float2(nx, ny);
              spv[gg] = sp;
              nzv[gg] = (anz && nrows > 0) ? 1 : 0;
              flv[gg] += 2LL * nrows;
            } else {
              nzv[gg] = 0;
            }
          }
        }
      };
      // the iterate goes to TMEM (asynchronous stores, drained after the aggregation barrier) as soon as this
      // warp's refresh is done: the weights are then formed with the registers free (every slot load of four
      // rows in flight), and the stores drain under the weights phase
      auto park = [&]() {
        float f0[16], f1[16];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          f0[2 * k] = m0[k].x; f0[2 * k + 1] = m0[k].y;
          f1[2 * k] = m0[k + 8].x; f1[2 * k + 1] = m0[k + 8].y;
        }
        tmem::st16(my_tmem, f0);
        tmem::st16(my_tmem + 16, f1);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          f0[2 * k] = m1[k].x; f0[2 * k + 1] = m1[k].y;
          f1[2 * k] = m1[k + 8].x; f1[2 * k + 1] = m1[k + 8].y;
        }
        tmem::st16(my_tmem + 32, f0);
        tmem::st16(my_tmem + 48, f1);
      };
      // aggregated projection (solvers.py:257-309): m parked in TMEM while y = sum phi h
      // (ascending rows) occupies the registers
      auto aggregate = [&](const int* ptr, const int* spl, const int2* L, int nrows, int span, bool dense, bool mark_done,
                           long long ycost) {
        if constexpr (PAR_W) reduce_weights(nrows);
#pragma unroll
        for (int k = 0; k < E; ++k) m0[k] = m1[k] = make_float2(0.f, 0.f);  // registers now hold y
        auto agg_entry = [&](auto jr, int2 e) {  // y += phi_i h_i on the entry's j range
          constexpr int J0 = decltype(jr)::lo, J1 = decltype(jr)::hi;
          const int i = e.x >> 20;
          KZ_CHECK(i < K && (e.x & 0xFFFFF) + CH <= pl.hcap, "wide: aggregated piece inside H");
          const T p0 = Phi[xs(i, g)], p1 = Phi[xs(i, g + 16)];
          const float4* hp = H4 + (((e.x & 0xFFFFF) + 2 * a) >> 1);
#pragma unroll
          for (int j = J0; j < J1; ++j) {
            float4 h = hp[2 * j];
            const int k = 2 * j;
            m0[k] = cfma(p0, make_float2(h.x, h.y), m0[k]);
            m0[k + 1] = cfma(p0, make_float2(h.z, h.w), m0[k + 1]);
            m1[k] = cfma(p1, make_float2(h.x, h.y), m1[k]);
            m1[k + 1] = cfma(p1, make_float2(h.z, h.w), m1[k + 1]);
          }
        };
        auto agg_seg = [&](auto jr, int q, const int q1) {
          for (; q + 1 < q1; q += 2) {  // two entries per trip: the next entry's loads overlap this one's FMAs
            const int2 ea = L[q], eb = L[q + 1];
            agg_entry(jr, ea);
            agg_entry(jr, eb);
          }
          if (q < q1) agg_entry(jr, L[q]);
        };
        agg_seg(JRange<0, 8>{}, ptr[w], spl[2 * w]);
        if constexpr (HALF) {
          agg_seg(JRange<0, 4>{}, spl[2 * w], spl[2 * w + 1]);
          agg_seg(JRange<4, 8>{}, spl[2 * w + 1], ptr[w + 1]);
        }
        float s0 = 0.f, s1 = 0.f;
#pragma unroll
        for (int k = 0; k < E; ++k) {
          s0 = fmaf(m0[k].x, m0[k].x, fmaf(m0[k].y, m0[k].y, s0));
          s1 = fmaf(m1[k].x, m1[k].x, fmaf(m1[k].y, m1[k].y, s1));
        }
        {  // ||y||^2 partial of this warp, stored [warp][rhs]: the warp's store and every lane-over-rhs read of
           // the step lengths below are bank-conflict free ([rhs][warp] with 16 warps put the 16 rhs of an LDS.128
           // on two 16-byte bank groups: 8-way conflicts in every thread's 8 loads)
          const float sd = a ? s0 : s1;
          const float rv = __shfl_xor_sync(FULL, sd, 16);
          Dp[w * G + g + 16 * a] = (a ? s1 : s0) + rv;
        }
        KZ_WSTAMP_IF(5);
        __syncthreads();
        KZ_PHASE();
        tmem::wait_st();
        KZ_PHASE();  // [timing] TMEM store drain
        float f0[16], f1[16];
        tmem::ld16(my_tmem, f0);  // the parked iterate streams in while the step lengths are formed
        tmem::ld16(my_tmem + 16, f1);
        KZ_PHASE();  // [timing] TMEM load issue
        // step length of this lane's own rhs g + 16 a (fixed-order pairwise sum of the warps' ||y||^2 partials: the
        // same value in every warp), the partner lane's by one exchange
        auto gamma_of = [&](int rr, bool& step) -> T {
          step = false;
          if (!nzv[rr]) return make_float2(0.f, 0.f);
          const float* dp = Dp + rr;
          float den;
          if (W == 16) {
            float u[16];
#pragma unroll
            for (int ww = 0; ww < 16; ++ww) u[ww] = dp[ww * G];
            den = ((u[0] + u[1]) + (u[2] + u[3]) + ((u[4] + u[5]) + (u[6] + u[7]))) +
                  ((u[8] + u[9]) + (u[10] + u[11]) + ((u[12] + u[13]) + (u[14] + u[15])));
          } else {
            den = 0.f;
            for (int ww = 0; ww < W; ++ww) den += dp[ww * G];
          }
          den = fmaf(regf, spv[rr], den);
          if (den == 0.f) return make_float2(0.f, 0.f);
          step = true;
          T nm = numv[rr];
          return make_float2(nm.x / den, nm.y / den);
        };
        bool st_own;
        const T gm_own = gamma_of(g + 16 * a, st_own);
        const T gm_oth = make_float2(__shfl_xor_sync(FULL, gm_own.x, 16), __shfl_xor_sync(FULL, gm_own.y, 16));
        const bool st_oth = __shfl_xor_sync(FULL, (int)st_own, 16) != 0;
        const bool st0 = a ? st_oth : st_own, st1 = a ? st_own : st_oth;
        const T gm0 = a ? gm_oth : gm_own, gm1 = a ? gm_own : gm_oth;
        KZ_WSTAMP_IF(6);
        KZ_PHASE();  // [timing] step lengths
        {
          tmem::wait_ld();
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            T o0 = make_float2(f0[2 * k], f0[2 * k + 1]), o1 = make_float2(f1[2 * k], f1[2 * k + 1]);
            m0[k] = st0 ? cfma(gm0, m0[k], o0) : o0;
            m0[k + 8] = st0 ? cfma(gm0, m0[k + 8], o1) : o1;
          }
          tmem::ld16(my_tmem + 32, f0);
          tmem::ld16(my_tmem + 48, f1);
          tmem::wait_ld();
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            T o0 = make_float2(f0[2 * k], f0[2 * k + 1]), o1 = make_float2(f1[2 * k], f1[2 * k + 1]);
            m1[k] = st1 ? cfma(gm1, m1[k], o0) : o0;
            m1[k + 8] = st1 ? cfma(gm1, m1[k + 8], o1) : o1;
          }
        }
        KZ_WSTAMP_IF(7);
        KZ_PHASE();  // [timing] iterate reload + update
        // q += gamma phi over the aggregated rows is left pending (flag in sel, length in gam): the next weights
        // pass applies it row by row where it loads q_i anyway, flush_q below after the last iteration
        if (w == 0) {
          sel[lane] = (a ? st1 : st0) && g0 + lane < K ? 1 : 0;
          gam[lane] = a ? gm1 : gm0;
        }
        KZ_PHASE();  // [timing] coefficient update
        // bookkeeping once per rhs (warp 0: lane = rhs slot)
        if (w == 0 && g0 + lane < K && !donev[lane]) {
          const bool st = a ? st1 : st0;
          const int n = nrows;
          if (!nzv[lane]) {
            noopv[lane] += 1;
            if (mark_done) donev[lane] = 1;
          } else {
            long long f = 6LL * n + 2LL * max(n - 1, 0) + ycost + 4LL * span + 3LL * n + 2;
            if (!st) {
              noopv[lane] += 1;
              if (mark_done) donev[lane] = 1;
            } else {
              f += 2 + 8LL * span + 8LL * n;
              if (SCH == KZ_AHK) itv[lane] += 1;
            }
            flv[lane] += f;
          }
        }
        KZ_WSTAMP_IF(8);
        (void)dense;
      };

      if constexpr (SCH == KZ_AHK) {
        refresh_list(lptr, lspl, lst);
        park();
        if (tid < G && g0 + tid < K && !donev[tid]) flv[tid] += dense_refresh;
        __syncthreads();
        KZ_PHASE();
        if constexpr (PAR_W) weights(0); else weights_rhs(0, K);
        __syncthreads();
        KZ_PHASE();
        aggregate(lptr, lspl, lst, K, Nt, true, true, 6LL * Nt * K + 2LL * Nt * max(K - 1, 0));
      } else {
        // exact block projection on the orthogonal group O (solvers.py:312-332)
        // the few O pieces of this chunk (disjoint VRs: one or two) in one compact loop -- a half piece taken as a
        // whole chunk adds its zero padding, which is exact -- instead of another copy of the unrolled refresh
        // (28 KB less code in the loop body: every phase of the iteration runs ~3% faster, instruction fetch)
        for (int q = optr[w]; q < optr[w + 1]; ++q) {
          const int2 e0 = olst[q];
          Ps[pslot(e0.y)] = dot_part(JRange<0, 8>{}, e0.x & 0xFFFFF);
        }
        KZ_WSTAMP_IF(1);
        __syncthreads();
        KZ_PHASE();
        for (int k = w; k < (int)misc[1]; k += W) {  // warp k: O row k, lanes over the rhs
          const int i = orow[k], rr = lane;
          if (g0 + rr >= K) continue;
          const T r = resid(i, rr);
          const T gm = make_float2(r.x / en[i], r.y / en[i]);
          const T q = Qs[xs(i, rr)];
          Qs[xs(i, rr)] = make_float2(q.x + gm.x, q.y + gm.y);
          Phi[xs(i, rr)] = gm;
        }
        if (tid < G && g0 + tid < K) flv[tid] += 2 * costO + (nN ? costN + 4LL * nN : 0);
        KZ_WSTAMP_IF(2);
        __syncthreads();
        KZ_PHASE();
        for (int q = optr[w]; q < optr[w + 1]; ++q) {
          const int i = olst[q].x >> 20;
          project(m0, i, Phi[xs(i, g)]);
          project(m1, i, Phi[xs(i, g + 16)]);
        }
        if (nN > 0) {
          refresh_list(nptr, nspl, nlst);
          park();
          KZ_WSTAMP_IF(3);
          __syncthreads();
          KZ_PHASE();
          if constexpr (PAR_W) weights(2); else weights_rhs(2, nN);
          KZ_WSTAMP_IF(4);
          __syncthreads();
          KZ_PHASE();
          aggregate(nptr, nspl, nlst, nN, unionN, false, false, costN);
        }
        if (tid < G && g0 + tid < K) itv[tid] += 1;
      }
      __syncthreads();  // bookkeeping visible before the all-done test
      KZ_PHASE();
    }
    if constexpr (NM) {
      // run_precoding's check (solvers.py:593-603): f_now = cols / ||cols||, err = ||f_ref - f_now|| / ||f_ref||,
      // the loop leaves at err < eps, then at the cap or when every rhs is done.  Both norms are fp64 sums of the
      // fp32 iterate (products exact in fp64), reduced per CTA in a fixed order and summed over the cluster in
      // rank order, so every CTA takes the same decision
      __syncthreads();  // this iteration's done flags and flop counts are visible
      double c2 = 0.0;
#pragma unroll
      for (int k = 0; k < E; ++k) {
        c2 = fma((double)m0[k].x, (double)m0[k].x, fma((double)m0[k].y, (double)m0[k].y, c2));
        c2 = fma((double)m1[k].x, (double)m1[k].x, fma((double)m1[k].y, (double)m1[k].y, c2));
      }
      const double cs = cta_sum_d(c2, red, w, lane, W);
      int nd = 0;
      long long fs = 0;
      if (tid < ngroups)
        for (int gg = 0; gg < G; ++gg)
          if (g0 + gg < K) {
            nd += donev[gg];
            fs += flv[gg];
          }
      double C;
      nmx_round1(nms, t, grp, ngroups, tid, cs, nd, fs, C, nd, fs);
      double err = 0.0;
      if (need_err) {
        const double mn = sqrt(C), inv = mn > 0.0 ? 1.0 / mn : 1.0;
        double d2 = 0.0;
        const double2* fr = reinterpret_cast<const double2*>(fref) + (size_t)(w * CH + 2 * a) * K + g0 + g;
        const bool v0 = g0 + g < K, v1 = g0 + g + 16 < K;  // rhs slots past K (ragged last group) hold m = 0
#pragma unroll 4
        for (int k = 0; k < E; ++k) {
          const size_t o = (size_t)(4 * (k >> 1) + (k & 1)) * K;
          const double2 f0 = v0 ? __ldg(fr + o) : make_double2(0.0, 0.0);
          const double2 f1 = v1 ? __ldg(fr + o + 16) : make_double2(0.0, 0.0);
          const double dx0 = fma(-(double)m0[k].x, inv, f0.x), dy0 = fma(-(double)m0[k].y, inv, f0.y);
          const double dx1 = fma(-(double)m1[k].x, inv, f1.x), dy1 = fma(-(double)m1[k].y, inv, f1.y);
          d2 = fma(dx0, dx0, fma(dy0, dy0, d2));
          d2 = fma(dx1, dx1, fma(dy1, dy1, d2));
        }
        err = sqrt(nmx_round2(nms, grp, ngroups, tid, cta_sum_d(d2, red, w, lane, W))) / fref_norm;
      }
      if (grp == 0 && tid == 0 && t - 1 < p.O.trace_cap) {
        if (p.O.nmse_trace) p.O.nmse_trace[(size_t)b * p.O.trace_cap + t - 1] = err;
        if (p.O.flops_trace) p.O.flops_trace[(size_t)b * p.O.trace_cap + t - 1] = fs;
      }
      conv = p.eps > 0.0 && err < p.eps;
      if (conv || nd == K) break;
    } else {
      bool all_done = true;
      for (int gg = 0; gg < G; ++gg)
        if (!donev[gg]) all_done = false;
      if (all_done) break;
    }
    // next iteration's writers of sel/gam run after the refresh barrier: no extra barrier needed
  }
  const int t_end = t > p.T ? p.T : t;
  __syncthreads();
  KZ_PHASE();
  if constexpr (AGG) {  // the last aggregated step's pending q += gamma phi
    if (sel[lane] > 0 && g0 + lane < K) {
      const T gq = gam[lane];
      for (int e = tid; e < K * G; e += nthr) {
        const int i = e / G;
        if (SCH == KZ_VR_OAHK && inset[i] != 2) continue;
        Qs[xs(i, lane)] = cfma(gq, Phi[xs(i, lane)], Qs[xs(i, lane)]);
      }
    }
    __syncthreads();
  }
  if constexpr (AGG) {
    tmem::fence_after();
    if (w == 0) tmem::dealloc(misc[0], 256);
  }

  // ------------------------------------------------------------------ outputs
  if (tid == 0) p.tstop[blockIdx.x] = t_end | (conv ? KZ_TSTOP_CONV : 0);
  KZ_TDUMP((long long*)((char*)p.tstop + ((size_t)p.P.n_systems * p.P.n_users * 4 + 7) / 8 * 8));
  auto store_m = [&](const T (&mr)[E], int r) {
    const int c = g0 + g + 16 * r;
    if (c >= K || !p.O.iterates) return;
    T* M = (T*)p.O.iterates + ((size_t)b * K + c) * Nt + w * CH;
#pragma unroll
    for (int k = 0; k < E; ++k) M[4 * (k >> 1) + 2 * a + (k & 1)] = mr[k];
  };
  store_m(m0, 0);
  store_m(m1, 1);
  T* vout = (T*)p.O.v;
  for (int e = tid; e < K * G; e += nthr) {
    int i = e / G, gg = e % G;
    if (g0 + gg < K) vout[((size_t)b * K + i) * K + g0 + gg] = Qs[xs(i, gg)];
  }
  for (int gg = tid; gg < G; gg += nthr) {
    int c = g0 + gg;
    if (c >= K) continue;
    size_t r = (size_t)b * K + c;
    if (p.O.iters) p.O.iters[r] = itv[gg];
    if (p.O.converged) p.O.converged[r] = 0;
    if (p.O.done) p.O.done[r] = donev[gg] ? 1 : 0;
    if (p.O.noop_steps) p.O.noop_steps[r] = noopv[gg];
    if (p.O.flops) p.O.flops[r] = flv[gg];
  }
}

inline size_t wide_smem_bytes(const kz_problem& P, int* S_out, int* hcap_out) {
  const int K = P.n_users;
  const int S = (P.max_support + wide::CH - 2) / wide::CH + 1;  // chunks a row can touch
  const int hcap = K * (S * wide::CH + wide::HSKEW);
  *S_out = S;
  *hcap_out = hcap;
  return wide::plan(K, P.n_antennas, S, hcap).total;
}

template <int SCH, bool NM>
inline int wide_launch(const kz_problem& P, const kz_rng& R, const kz_out& O, int T_iters, const double* f_ref,
                       double eps, char* ws, int32_t* tstop, size_t smem, int S, int hcap, cudaStream_t s) {
  LsArgs a;
  a.P = P;
  a.R = R;
  a.O = O;
  a.T = T_iters;
  a.S = S;
  a.hcap = hcap;
  a.ws = ws;
  a.L = gen_layout(P.n_systems, P.n_users, P.n_antennas, P.dtype);
  a.tstop = tstop;
  a.f_ref = f_ref;
  a.eps = eps;
  a.bulk = bulk_staging_ok(P);
  const int groups = (P.n_users + wide::G - 1) / wide::G;
  auto kern = kz_wide_kernel<SCH, NM>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return -1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(P.n_systems * groups));
  cfg.blockDim = dim3((unsigned)P.n_antennas);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  if (NM) {  // the system's CTAs form one cluster (NMSE partials over DSMEM)
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)groups;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) != cudaSuccess || nclusters < 1) {
      cudaGetLastError();
      return 0;
    }
    if (getenv("KZ_VERBOSE"))
      fprintf(stderr, "[kz wide nmse] cluster %d smem %zu: max active clusters %d\n", groups, smem, nclusters);
  }
  if (g_dry_launch) return 1;
  note_tma(a.bulk);
  if (cudaLaunchKernelEx(&cfg, kern, a) != cudaSuccess) return -1;
  kz_lockstep_finalize<<<(P.n_systems + 127) / 128, 128, 0, s>>>(tstop, groups, P.n_systems, O.n_outer,
                                                                  O.sys_converged);
  return 1;
}

// 1 launched, 0 not eligible / not a single-row scheme, -1 failure.  nm: NMSE-stopped / traced lockstep run
// (f_ref, eps; T = the cap)
inline int wide_dispatch(const kz_problem& P, int scheme, const kz_rng& R, const kz_out& O, int T_iters, bool nm,
                         const double* f_ref, double eps, char* ws, int32_t* tstop, int maxsm, cudaStream_t s) {
  if (P.dtype != KZ_C64 || P.n_antennas % wide::CH != 0 || P.n_users < 17 || P.n_users > 128) return 0;
  int S, hcap;
  size_t smem = wide_smem_bytes(P, &S, &hcap);
  if ((int)smem > maxsm) return 0;
#define KZ_WIDE_CASE(SC)                                                                                    \
  case SC:                                                                                                  \
    return nm ? wide_launch<SC, true>(P, R, O, T_iters, f_ref, eps, ws, tstop, smem, S, hcap, s)           \
              : wide_launch<SC, false>(P, R, O, T_iters, f_ref, eps, ws, tstop, smem, S, hcap, s);
  switch (scheme) {
    KZ_WIDE_CASE(KZ_URK)
    KZ_WIDE_CASE(KZ_SWOR_ERK)
    KZ_WIDE_CASE(KZ_GK)
    KZ_WIDE_CASE(KZ_GRK)
    KZ_WIDE_CASE(KZ_VR_OGRK)
    KZ_WIDE_CASE(KZ_AHK)
    KZ_WIDE_CASE(KZ_VR_OAHK)
  }
#undef KZ_WIDE_CASE
  return 0;
}

}  // namespace kz
