// Load-balanced register-resident lockstep kernel (complex64 throughput path).
//
// Same CTA mapping as kz_solve_lockstep.cuh (one system x G = 16 rhs, the
// iterate m in registers, rows h_i in shared memory), with three changes
// driven by the ncu profile of the chunked kernel (profiles/r01_*):
//   * Work balance.  The antenna axis is cut into 16-antenna PIECES and each
//     warp owns two of them, assigned per system by longest-processing-time
//     on the number of rows overlapping each piece.  With contiguous chunks
//     the busiest warp carried 1.59x the mean row count (the trapezoidal VR
//     coverage plus clustering) and the CTA barriers turned that into ~40%
//     stall; LPT pieces bring it to ~1.14x.
//   * No predicates.  Rows are stored zero-padded to whole pieces, so every
//     (row, piece) product is a fixed 8-element FMA block fed by broadcast
//     LDS.128 loads; the padding contributes exact zeros.
//   * Fewer barriers.  Residual finalisation (sum of the per-warp partial
//     slots, fixed order => deterministic) is fused into the per-rhs
//     selection / weighting warp, and the aggregated step computes its step
//     length redundantly per thread, so GRK-type schemes use 2 CTA barriers
//     per iteration and AHK-type schemes 3.
// Reference semantics are those of kz_solve_lockstep.cuh (solvers.py:382-423).
#pragma once

#include "kz_common.cuh"
#include "kz_solve_generic.cuh"

namespace kz {

namespace bal {

constexpr int G = 16;          // rhs per CTA
constexpr int A = 2;           // lanes per rhs (antenna split)
constexpr int PS = 16;         // piece size (antennas)
constexpr int PPW = 2;         // pieces per warp
constexpr int EPP = PS / A;    // elements per piece per thread (8)
constexpr int NPT = PPW * EPP; // iterate entries per thread (16)

struct Plan {
  int K, W, NP, SL, hcap;
  size_t rowS, rowL, rowB, p0, p1, en, cost, cmask, nsl, slotOf, inset, pload, pbase, lall, lo, ln, lcnt, H, P, Q, R, Dp,
      sel, gam, num, sp, nz, done, iters, noop, flops, prev, pool, poolcnt, misc, total;
};

__host__ __device__ inline size_t al(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline Plan plan(int K, int Nt, int SL, int hcap) {
  Plan p;
  p.K = K;
  p.W = Nt / 32;
  p.NP = Nt / PS;
  p.SL = SL;
  p.hcap = hcap;
  const int KW = (K + 31) / 32;
  size_t o = 0;
  p.rowS = o; o = al(o + 4 * K);
  p.rowL = o; o = al(o + 4 * K);
  p.rowB = o; o = al(o + 4 * K);
  p.p0 = o; o = al(o + 4 * K);
  p.p1 = o; o = al(o + 4 * K);
  p.en = o; o = al(o + 8 * K);
  p.cost = o; o = al(o + 8 * K);
  p.cmask = o; o = al(o + 4 * (size_t)K * KW);
  p.nsl = o; o = al(o + 4 * K);
  p.slotOf = o; o = al(o + (size_t)K * p.W);
  p.inset = o; o = al(o + K);
  p.pload = o; o = al(o + 4 * p.NP);
  p.pbase = o; o = al(o + 4 * p.W * PPW);
  p.lall = o; o = al(o + 4 * (size_t)p.W * K);
  p.lo = o; o = al(o + 4 * (size_t)p.W * K);
  p.ln = o; o = al(o + 4 * (size_t)p.W * K);
  p.lcnt = o; o = al(o + 4 * 3 * p.W);
  p.H = o; o = al(o + 8 * (size_t)hcap);
  size_t psz = 8 * (size_t)K * SL * G;
  p.P = o; o = al(o + (psz > 8 * (size_t)K * G ? psz : 8 * (size_t)K * G));
  p.Q = o; o = al(o + 8 * (size_t)K * G);
  p.R = o; o = al(o + 8 * (size_t)K * G);
  p.Dp = o; o = al(o + 4 * (size_t)p.W * G);
  p.sel = o; o = al(o + 4 * G);
  p.gam = o; o = al(o + 8 * G);
  p.num = o; o = al(o + 8 * G);
  p.sp = o; o = al(o + 4 * G);
  p.nz = o; o = al(o + 4 * G);
  p.done = o; o = al(o + 4 * G);
  p.iters = o; o = al(o + 4 * G);
  p.noop = o; o = al(o + 4 * G);
  p.flops = o; o = al(o + 8 * G);
  p.prev = o; o = al(o + 4 * G);
  p.pool = o; o = al(o + 4 * (size_t)G * KW);
  p.poolcnt = o; o = al(o + 4 * G);
  p.misc = o; o = al(o + 64);
  p.total = o;
  return p;
}

}  // namespace bal

template <int SCH>
__global__ void __launch_bounds__(512, 1) kz_balanced_kernel(LsArgs p) {
  using namespace bal;
  using T = float2;
  constexpr bool PER_LANE_ROW = SCH == KZ_URK || SCH == KZ_SWOR_ERK;
  constexpr bool DENSE_FORM = SCH == KZ_GK || SCH == KZ_GRK || SCH == KZ_AHK;

  extern __shared__ __align__(16) unsigned char sm[];
  const int K = p.P.n_users, Nt = p.P.n_antennas;
  const int ngroups = (K + G - 1) / G;
  const int b = blockIdx.x / ngroups, grp = blockIdx.x % ngroups, g0 = grp * G;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31, g = lane % G, a = lane / G;
  const int nthr = blockDim.x;
  const Plan pl = plan(K, Nt, p.S, p.hcap);
  const int W = pl.W, NP = pl.NP, SL = pl.SL, KW = (K + 31) / 32;

  int* rowS = (int*)(sm + pl.rowS);
  int* rowL = (int*)(sm + pl.rowL);
  int* rowB = (int*)(sm + pl.rowB);
  int* p0 = (int*)(sm + pl.p0);
  int* p1 = (int*)(sm + pl.p1);
  double* en = (double*)(sm + pl.en);
  long long* cost = (long long*)(sm + pl.cost);
  uint32_t* cmask = (uint32_t*)(sm + pl.cmask);
  int* nsl = (int*)(sm + pl.nsl);
  uint8_t* slotOf = (uint8_t*)(sm + pl.slotOf);
  uint8_t* inset = (uint8_t*)(sm + pl.inset);
  int* pload = (int*)(sm + pl.pload);
  int* pbase = (int*)(sm + pl.pbase);
  int* lall = (int*)(sm + pl.lall);
  int* lo_ = (int*)(sm + pl.lo);
  int* ln_ = (int*)(sm + pl.ln);
  int* lcnt = (int*)(sm + pl.lcnt);
  T* Hs = (T*)(sm + pl.H);
  T* Ps = (T*)(sm + pl.P);
  T* Phi = Ps;
  T* Qs = (T*)(sm + pl.Q);
  T* Rs = (T*)(sm + pl.R);
  float* Dp = (float*)(sm + pl.Dp);
  int* sel = (int*)(sm + pl.sel);
  T* gam = (T*)(sm + pl.gam);
  T* numv = (T*)(sm + pl.num);
  float* spv = (float*)(sm + pl.sp);
  int* nzv = (int*)(sm + pl.nz);
  int* donev = (int*)(sm + pl.done);
  int* itv = (int*)(sm + pl.iters);
  int* noopv = (int*)(sm + pl.noop);
  long long* flv = (long long*)(sm + pl.flops);
  int* prevv = (int*)(sm + pl.prev);
  uint32_t* poolv = (uint32_t*)(sm + pl.pool);
  int* poolcnt = (int*)(sm + pl.poolcnt);
  int* misc = (int*)(sm + pl.misc);

  const double reg = p.P.reg[b];
  const float regf = (float)reg;
  const T* heff = (const T*)p.P.heff;

  // ------------------------------------------------------------------ setup
  for (int i = tid; i < K; i += nthr) {
    size_t r = (size_t)b * K + i;
    int sg = p.P.row_seg_ptr[r];
    int s = p.P.seg_start[sg], L = p.P.seg_len[sg];
    rowS[i] = s;
    rowL[i] = L;
    p0[i] = s / PS;
    p1[i] = (s + L - 1) / PS;
    en[i] = p.P.row_energy[r];
    inset[i] = 0;
  }
  if (tid == 0) {
    int no = 0, nn = 0;
    if (p.P.orth_ptr) {
      no = p.P.orth_ptr[b + 1] - p.P.orth_ptr[b];
      nn = p.P.non_ptr[b + 1] - p.P.non_ptr[b];
    }
    misc[1] = no;
    misc[2] = nn;
    misc[3] = p.P.non_union_size ? p.P.non_union_size[b] : 0;
  }
  __syncthreads();
  if (p.P.orth_ptr) {  // 1 = orthogonal group O, 2 = non-orthogonal N
    for (int q = p.P.orth_ptr[b] + tid; q < p.P.orth_ptr[b + 1]; q += nthr) inset[p.P.orth_idx[q]] = 1;
    for (int q = p.P.non_ptr[b] + tid; q < p.P.non_ptr[b + 1]; q += nthr) inset[p.P.non_idx[q]] = 2;
  }
  for (int pc = tid; pc < NP; pc += nthr) {
    int c = 0;
    for (int i = 0; i < K; ++i) c += (p0[i] <= pc && pc <= p1[i]);
    pload[pc] = c;
  }
  __syncthreads();
  if (tid == 0) {
    // row bases (whole pieces, zero padded)
    int base = 0;
    for (int i = 0; i < K; ++i) {
      rowB[i] = base;
      base += (p1[i] - p0[i] + 1) * PS;
    }
    // LPT: pieces by descending load (ties: lower index), each to the least-loaded warp with room
    int order[64];
    for (int pc = 0; pc < NP; ++pc) order[pc] = pc;
    for (int x = 1; x < NP; ++x) {
      int v = order[x], y = x - 1;
      while (y >= 0 && (pload[order[y]] < pload[v] || (pload[order[y]] == pload[v] && order[y] > v))) {
        order[y + 1] = order[y];
        --y;
      }
      order[y + 1] = v;
    }
    int wl[32], wn[32];
    for (int ww = 0; ww < W; ++ww) wl[ww] = wn[ww] = 0;
    for (int x = 0; x < NP; ++x) {
      int best = -1;
      for (int ww = 0; ww < W; ++ww)
        if (wn[ww] < PPW && (best < 0 || wl[ww] < wl[best])) best = ww;
      pbase[best * PPW + wn[best]] = order[x] * PS;
      wl[best] += pload[order[x]];
      wn[best] += 1;
    }
  }
  __syncthreads();
  // per row: owner warps of its pieces -> slot numbers (ascending warp id)
  for (int i = tid; i < K; i += nthr) {
    uint32_t own = 0;
    for (int ww = 0; ww < W; ++ww)
      for (int q = 0; q < PPW; ++q) {
        int pc = pbase[ww * PPW + q] / PS;
        if (p0[i] <= pc && pc <= p1[i]) own |= 1u << ww;
      }
    int n = 0;
    for (int ww = 0; ww < W; ++ww) {
      slotOf[i * W + ww] = (own >> ww) & 1u ? (uint8_t)n : (uint8_t)255;
      n += (own >> ww) & 1u;
    }
    nsl[i] = n;
  }
  __syncthreads();
  // per-warp row lists (ascending rows): entry = row | piece-mask << 16 | slot << 24
  {
    int pcs[PPW];
    for (int q = 0; q < PPW; ++q) pcs[q] = pbase[w * PPW + q] / PS;
    int na = 0, no = 0, nn = 0;
    for (int base = 0; base < K; base += 32) {
      int i = base + lane;
      int mask = 0;
      if (i < K)
        for (int q = 0; q < PPW; ++q) mask |= (p0[i] <= pcs[q] && pcs[q] <= p1[i]) << q;
      int ent = i | (mask << 16) | ((i < K ? slotOf[i * W + w] : 0) << 24);
      unsigned bal_a = __ballot_sync(FULL, mask != 0);
      unsigned bal_o = __ballot_sync(FULL, mask != 0 && inset[i < K ? i : 0] == 1);
      unsigned bal_n = __ballot_sync(FULL, mask != 0 && inset[i < K ? i : 0] == 2);
      unsigned lt = (1u << lane) - 1;
      if (mask) {
        lall[w * K + na + __popc(bal_a & lt)] = ent;
        if (inset[i] == 1) lo_[w * K + no + __popc(bal_o & lt)] = ent;
        if (inset[i] == 2) ln_[w * K + nn + __popc(bal_n & lt)] = ent;
      }
      na += __popc(bal_a);
      no += __popc(bal_o);
      nn += __popc(bal_n);
    }
    if (lane == 0) {
      lcnt[w * 3 + 0] = na;
      lcnt[w * 3 + 1] = no;
      lcnt[w * 3 + 2] = nn;
    }
  }
  // rows -> shared memory, zero padded to whole pieces: antenna n of row i at Hs[rowB_i + n - PS*p0_i]
  for (int i = 0; i < K; ++i) {
    const T* src = heff + p.P.row_val_ptr[(size_t)b * K + i];
    const int s = rowS[i], L = rowL[i], lo = p0[i] * PS, span = (p1[i] - p0[i] + 1) * PS;
    T* dst = Hs + rowB[i];
    for (int j = tid; j < span; j += nthr) {
      int n = lo + j;
      dst[j] = (n >= s && n < s + L) ? src[n - s] : make_float2(0.f, 0.f);
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
    Qs[e] = make_float2(0.f, 0.f);
    Rs[e] = make_float2(i == g0 + gg ? 1.f : 0.f, 0.f);
  }
  for (int gg = tid; gg < G; gg += nthr) {
    donev[gg] = (g0 + gg < K) ? 0 : 1;
    itv[gg] = 0;
    noopv[gg] = 0;
    flv[gg] = 0;
    prevv[gg] = -1;
    poolcnt[gg] = 0;
    sel[gg] = -1;
    nzv[gg] = 0;
  }
  __syncthreads();
  const int nN = misc[2], unionN = misc[3];
  long long costO = 0, costN = 0;
  for (int i = 0; i < K; ++i) {
    if (inset[i] == 1) costO += 8LL * rowL[i] + 4;
    if (inset[i] == 2) costN += 8LL * rowL[i];
  }
  int pb[PPW];
#pragma unroll
  for (int q = 0; q < PPW; ++q) pb[q] = pbase[w * PPW + q];

  T m[NPT];
#pragma unroll
  for (int k = 0; k < NPT; ++k) m[k] = make_float2(0.f, 0.f);
  // antenna of element e (0..EPP-1) of piece q for this thread: pair-interleaved over the a-lanes
  auto ant = [&](int q, int e) { return pb[q] + (e >> 1) * (2 * A) + 2 * a + (e & 1); };
  auto rowp = [&](int i) -> const T* { return Hs + rowB[i] - PS * p0[i]; };

  // partial conj(h_i) . m over the pieces in `mask` (rows zero padded => no predicates)
  auto partial = [&](int i, int mask) -> T {
    const T* hp = rowp(i);
    T c0 = make_float2(0.f, 0.f), c1 = make_float2(0.f, 0.f);
#pragma unroll
    for (int q = 0; q < PPW; ++q) {
      if (!((mask >> q) & 1)) continue;
#pragma unroll
      for (int e = 0; e < EPP; e += 2) {
        float4 h = *reinterpret_cast<const float4*>(hp + ant(q, e));
        c0 = cfma_conj(make_float2(h.x, h.y), m[q * EPP + e], c0);
        c1 = cfma_conj(make_float2(h.z, h.w), m[q * EPP + e + 1], c1);
      }
    }
    T acc = make_float2(c0.x + c1.x, c0.y + c1.y);
    acc.x += __shfl_xor_sync(FULL, acc.x, G);
    acc.y += __shfl_xor_sync(FULL, acc.y, G);
    return acc;
  };
  // refresh partials of a warp list into P[i][slot][g]; two rows in flight for ILP
  auto refresh = [&](const int* lst, int n) {
    int q = 0;
    for (; q + 1 < n; q += 2) {
      int e0 = lst[q], e1 = lst[q + 1];
      T v0 = partial(e0 & 0xffff, (e0 >> 16) & 0xff);
      T v1 = partial(e1 & 0xffff, (e1 >> 16) & 0xff);
      if (a == 0) {
        Ps[((size_t)(e0 & 0xffff) * SL + (e0 >> 24)) * G + g] = v0;
        Ps[((size_t)(e1 & 0xffff) * SL + (e1 >> 24)) * G + g] = v1;
      }
    }
    if (q < n) {
      int e0 = lst[q];
      T v0 = partial(e0 & 0xffff, (e0 >> 16) & 0xff);
      if (a == 0) Ps[((size_t)(e0 & 0xffff) * SL + (e0 >> 24)) * G + g] = v0;
    }
  };
  // residual of row i for rhs slot gg from the partial slots (fixed order)
  auto resid = [&](int i, int gg) -> T {
    const T* pp = Ps + (size_t)i * SL * G + gg;
    T dot = make_float2(0.f, 0.f);
    for (int s = 0; s < nsl[i]; ++s) {
      T v = pp[(size_t)s * G];
      dot.x += v.x;
      dot.y += v.y;
    }
    T q = Qs[i * G + gg];
    const int c = g0 + gg;
    if (DENSE_FORM) {
      T r = make_float2(-dot.x - q.x * regf, -dot.y - q.y * regf);
      if (i == c) r.x += 1.f;
      return r;
    } else {
      float tg = i == c ? 1.f : 0.f;
      return make_float2((tg - dot.x) - q.x * regf, (0.f - dot.y) - q.y * regf);
    }
  };
  auto draw_u = [&](int gg) -> double {
    int c = g0 + gg, d = itv[gg];
    if (p.R.kind == KZ_RNG_PHILOX) return philox_uniform(p.R.seed, (uint32_t)b, (uint32_t)c, (uint64_t)d);
    return p.R.uniforms[((size_t)b * K + c) * p.R.stream_len + d];
  };
  auto log_row = [&](int gg, int it, int i) {
    if (p.O.rows && it < p.O.rows_cap) p.O.rows[((size_t)b * K + g0 + gg) * p.O.rows_cap + it] = i;
  };
  auto take_step = [&](int gg, int i, T r, long long f) {
    T gm = make_float2(r.x / (float)en[i], r.y / (float)en[i]);
    Qs[i * G + gg] = make_float2(Qs[i * G + gg].x + gm.x, Qs[i * G + gg].y + gm.y);
    Rs[i * G + gg] = make_float2(0.f, 0.f);
    gam[gg] = gm;
    sel[gg] = i;
    log_row(gg, itv[gg], i);
    itv[gg] += 1;
    flv[gg] += f;
  };
  // m += gm * h_i on this thread's pieces overlapping row i (per-lane row)
  auto project_row = [&](int i, T gm) {
    const T* hp = rowp(i);
#pragma unroll
    for (int q = 0; q < PPW; ++q) {
      int pc = pb[q] / PS;
      if (pc < p0[i] || pc > p1[i]) continue;
#pragma unroll
      for (int e = 0; e < EPP; e += 2) {
        float4 h = *reinterpret_cast<const float4*>(hp + ant(q, e));
        m[q * EPP + e] = cfma(gm, make_float2(h.x, h.y), m[q * EPP + e]);
        m[q * EPP + e + 1] = cfma(gm, make_float2(h.z, h.w), m[q * EPP + e + 1]);
      }
    }
  };
  // greedy-weighted (GRK, Eq. 18) pick for rhs gg; lanes over rows; also finalises the
  // residuals it reads (all rows for grk, the coupled set of prev for vr-ogrk)
  auto finalize_rows = [&](int gg) {
    for (int i = lane; i < K; i += 32) {
      if constexpr (SCH == KZ_VR_OGRK) {
        int pr = prevv[gg];
        if (pr < 0 || !((cmask[pr * KW + (i >> 5)] >> (i & 31)) & 1u)) continue;
      }
      Rs[i * G + gg] = resid(i, gg);
    }
    __syncwarp();
  };
  auto pick_weighted = [&](int gg) -> int {
    float tot = 0.f;
    for (int i = lane; i < K; i += 32) {
      T r = Rs[i * G + gg];
      tot += r.x * r.x + r.y * r.y;
    }
    tot = warp_sum(tot);
    if (tot == 0.f) return -2;  // None: no draw consumed
    const float tau = (float)draw_u(gg) * tot;
    float carry = 0.f;
    int lastnz = -1;
    for (int base = 0; base < K; base += 32) {
      int i = base + lane;
      float v = 0.f;
      if (i < K) {
        T r = Rs[i * G + gg];
        v = r.x * r.x + r.y * r.y;
      }
      float sc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        float t2 = __shfl_up_sync(FULL, sc, o);
        if (lane >= o) sc += t2;
      }
      unsigned bal = __ballot_sync(FULL, i < K && v > 0.f && carry + sc > tau);
      if (bal) return base + __ffs(bal) - 1;
      unsigned nzb = __ballot_sync(FULL, i < K && v > 0.f);
      if (nzb) lastnz = base + 31 - __clz(nzb);
      carry += __shfl_sync(FULL, sc, 31);
    }
    return lastnz;
  };
  auto pick_max = [&](int gg) -> int {
    float best = -1.f;
    int bi = 0x7fffffff;
    bool any = false;
    for (int i = lane; i < K; i += 32) {
      T r = Rs[i * G + gg];
      float s = (r.x * r.x + r.y * r.y) / (float)en[i];
      if (s != 0.f) any = true;
      if (s > best) { best = s; bi = i; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      float ob = __shfl_xor_sync(FULL, best, o);
      int oi = __shfl_xor_sync(FULL, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    return __any_sync(FULL, any) ? bi : -2;
  };

  // aggregated step over the rows of set `setid` (0 = all, 2 = N) using the warp list `lst`:
  // finalise residuals + weights (warp per rhs), y = sum phi h (ascending rows), den, update.
  T y[NPT];
  auto aggregate = [&](int setid, const int* lst, int nl, int nrows, int span, bool dense, bool mark_done) {
    for (int gg = w; gg < G; gg += W) {
      if (g0 + gg >= K || donev[gg]) {
        if (lane == 0) nzv[gg] = 0;
        continue;
      }
      T num = make_float2(0.f, 0.f);
      float sp = 0.f;
      bool nz = false;
      for (int i = lane; i < K; i += 32) {
        if (setid != 0 && inset[i] != setid) continue;
        T r = resid(i, gg);
        T ph = make_float2(r.x / (float)en[i], r.y / (float)en[i]);
        Phi[i * G + gg] = ph;
        if (ph.x != 0.f || ph.y != 0.f) nz = true;
        num = cfma_conj(ph, r, num);
        sp += ph.x * ph.x + ph.y * ph.y;
      }
      num = warp_csum(num);
      sp = warp_sum(sp);
      nz = __any_sync(FULL, nz);
      if (lane == 0) {
        numv[gg] = num;
        spv[gg] = sp;
        nzv[gg] = (nz && nrows > 0) ? 1 : 0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NPT; ++k) y[k] = make_float2(0.f, 0.f);
    const bool act = nzv[g] != 0;
    for (int q = 0; q < nl; ++q) {
      int ent = lst[q], i = ent & 0xffff, mask = (ent >> 16) & 0xff;
      const T ph = Phi[i * G + g];
      const T* hp = rowp(i);
#pragma unroll
      for (int pq = 0; pq < PPW; ++pq) {
        if (!((mask >> pq) & 1)) continue;
#pragma unroll
        for (int e = 0; e < EPP; e += 2) {
          float4 h = *reinterpret_cast<const float4*>(hp + ant(pq, e));
          y[pq * EPP + e] = cfma(ph, make_float2(h.x, h.y), y[pq * EPP + e]);
          y[pq * EPP + e + 1] = cfma(ph, make_float2(h.z, h.w), y[pq * EPP + e + 1]);
        }
      }
    }
    float sy = 0.f;
#pragma unroll
    for (int k = 0; k < NPT; ++k) sy += y[k].x * y[k].x + y[k].y * y[k].y;
    sy += __shfl_xor_sync(FULL, sy, G);
    if (a == 0) Dp[w * G + g] = sy;
    __syncthreads();
    // step length (redundantly per thread; fixed summation order)
    float den = 0.f;
    for (int ww = 0; ww < W; ++ww) den += Dp[ww * G + g];
    den += regf * spv[g];
    const bool step = act && den != 0.f;
    if (step) {
      T nm = numv[g];
      T gm = make_float2(nm.x / den, nm.y / den);
#pragma unroll
      for (int k = 0; k < NPT; ++k) m[k] = cfma(gm, y[k], m[k]);
    }
    if (w == 0 && a == 0 && g0 + g < K && !donev[g]) {  // bookkeeping once per rhs
      const int n = nrows;
      if (!act) {
        noopv[g] += 1;
        if (mark_done) donev[g] = 1;
      } else {
        long long f = 6LL * n + 2LL * max(n - 1, 0);
        f += dense ? 6LL * Nt * n + 2LL * Nt * max(n - 1, 0) : (setid == 0 ? 0 : costN);
        f += 4LL * span + 3LL * n + 2;
        if (!step) {
          noopv[g] += 1;
          if (mark_done) donev[g] = 1;
        } else {
          f += 2 + 8LL * span + 8LL * n;
          itv[g] += (SCH == KZ_AHK) ? 1 : 0;
        }
        flv[g] += f;
      }
      flv[g] += 2LL * n;  // aggregation_weights
    }
    // q += gamma phi over the set rows (threads over (i, g) pairs)
    for (int e = tid; e < K * G; e += nthr) {
      int i = e / G, gg = e % G;
      if (setid != 0 && inset[i] != setid) continue;
      if (!nzv[gg] || g0 + gg >= K) continue;
      float d2 = 0.f;
      for (int ww = 0; ww < W; ++ww) d2 += Dp[ww * G + gg];
      d2 += regf * spv[gg];
      if (d2 == 0.f) continue;
      T nm = numv[gg];
      T gm = make_float2(nm.x / d2, nm.y / d2);
      Qs[e] = cfma(gm, Phi[e], Qs[e]);
    }
  };

  // ------------------------------------------------------------------ iterations
  const long long dense_refresh = 6LL * K * Nt + 2LL * K * (Nt + 1) + 2LL * K;
  const long long dense_rk = 2 + 8LL * Nt + 2;
  const int nall = lcnt[w * 3 + 0], nlo = lcnt[w * 3 + 1], nln = lcnt[w * 3 + 2];
  const int* Lall = lall + w * K;
  const int* Lo = lo_ + w * K;
  const int* Ln = ln_ + w * K;
  int t;
  for (t = 1; t <= p.T; ++t) {
    if constexpr (SCH == KZ_GRK || SCH == KZ_GK || SCH == KZ_VR_OGRK) {
      refresh(Lall, nall);
      __syncthreads();
      for (int gg = w; gg < G; gg += W) {
        if (g0 + gg >= K || donev[gg]) {
          if (lane == 0) sel[gg] = -1;
          continue;
        }
        finalize_rows(gg);
        long long f;
        int i;
        if constexpr (SCH == KZ_GK) {
          i = pick_max(gg);
          f = dense_refresh + 4LL * K;
        } else {
          i = pick_weighted(gg);
          f = (SCH == KZ_GRK ? dense_refresh : (prevv[gg] >= 0 ? cost[prevv[gg]] : 0)) + 4LL * K + 2;
        }
        if (lane == 0) {
          if (i < 0) {
            donev[gg] = 1;
            sel[gg] = -1;
            flv[gg] += f;
          } else {
            long long fr = SCH == KZ_VR_OGRK ? 2 + 8LL * rowL[i] + 2 : dense_rk;
            take_step(gg, i, Rs[i * G + gg], f + fr);
            if constexpr (SCH == KZ_VR_OGRK) prevv[gg] = i;
          }
        }
        __syncwarp();
      }
      __syncthreads();
      const int i = sel[g];
      if (i >= 0) project_row(i, gam[g]);
    } else if constexpr (PER_LANE_ROW) {
      for (int gg = tid; gg < G; gg += nthr) {
        if (g0 + gg >= K || donev[gg]) {
          sel[gg] = -1;
          continue;
        }
        int c = g0 + gg, d = itv[gg], i;
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
            if ((pbm[j >> 5] >> (j & 31)) & 1u) tot += en[j];
          double u = draw_u(gg) * tot, acc = 0.0;
          int last = -1;
          i = -1;
          for (int j = 0; j < K; ++j) {
            if (!((pbm[j >> 5] >> (j & 31)) & 1u)) continue;
            last = j;
            acc += en[j];
            if (acc > u) { i = j; break; }
          }
          if (i < 0) i = last;
          pbm[i >> 5] &= ~(1u << (i & 31));
          poolcnt[gg] -= 1;
        }
        sel[gg] = i;
        flv[gg] += f;
      }
      __syncthreads();
      {  // partial of each lane's own row on this warp's pieces
        const int i = sel[g];
        T v = make_float2(0.f, 0.f);
        int mask = 0;
        if (i >= 0)
          for (int q = 0; q < PPW; ++q) mask |= (p0[i] <= pb[q] / PS && pb[q] / PS <= p1[i]) << q;
        if (mask) {
          const T* hp = rowp(i);
#pragma unroll
          for (int q = 0; q < PPW; ++q) {
            if (!((mask >> q) & 1)) continue;
#pragma unroll
            for (int e = 0; e < EPP; e += 2) {
              float4 h = *reinterpret_cast<const float4*>(hp + ant(q, e));
              v = cfma_conj(make_float2(h.x, h.y), m[q * EPP + e], v);
              v = cfma_conj(make_float2(h.z, h.w), m[q * EPP + e + 1], v);
            }
          }
        }
        v.x += __shfl_xor_sync(FULL, v.x, G);
        v.y += __shfl_xor_sync(FULL, v.y, G);
        if (mask && a == 0) Ps[((size_t)i * SL + slotOf[i * W + w]) * G + g] = v;
      }
      __syncthreads();
      for (int gg = tid; gg < G; gg += nthr) {
        const int i = sel[gg];
        if (i < 0) continue;
        take_step(gg, i, resid(i, gg), 2 * (8LL * Nt + 4));
      }
      __syncthreads();
      const int i = sel[g];
      if (i >= 0) project_row(i, gam[g]);
    } else if constexpr (SCH == KZ_AHK) {
      refresh(Lall, nall);
      for (int gg = tid; gg < G; gg += nthr)
        if (g0 + gg < K && !donev[gg]) flv[gg] += dense_refresh;
      __syncthreads();
      aggregate(0, Lall, nall, K, Nt, true, true);
    } else {  // KZ_VR_OAHK
      refresh(Lo, nlo);
      __syncthreads();
      // exact block projection on O: residual -> gamma, q += gamma (thread per (row, rhs))
      for (int e = tid; e < K * G; e += nthr) {
        int i = e / G, gg = e % G;
        if (inset[i] != 1 || g0 + gg >= K) continue;
        T r = resid(i, gg);
        T gm = make_float2(r.x / (float)en[i], r.y / (float)en[i]);
        Qs[e] = make_float2(Qs[e].x + gm.x, Qs[e].y + gm.y);
        Rs[e] = make_float2(0.f, 0.f);
        Rs[e] = gm;  // gamma parked in R until the projection below (R is not read by vr-oahk)
      }
      if (w == 0 && a == 0 && g0 + g < K) flv[g] += 2 * costO;
      __syncthreads();
      for (int q = 0; q < nlo; ++q) {
        int i = Lo[q] & 0xffff;
        project_row(i, Rs[i * G + g]);
      }
      if (nN > 0) {
        refresh(Ln, nln);
        if (w == 0 && a == 0 && g0 + g < K) flv[g] += costN + 4LL * nN;
        __syncthreads();
        aggregate(2, Ln, nln, nN, unionN, false, false);
      }
      if (w == 0 && a == 0 && g0 + g < K) itv[g] += 1;
    }
    __syncthreads();
    bool all_done = true;
    for (int gg = 0; gg < G; ++gg)
      if (!donev[gg]) all_done = false;
    if (all_done) break;
  }
  const int t_end = t > p.T ? p.T : t;

  // ------------------------------------------------------------------ outputs
  if (tid == 0) p.tstop[blockIdx.x] = t_end;
  {
    const int c = g0 + g;
    if (c < K) {
      T* M = (T*)(p.ws + p.L.M) + ((size_t)b * K + c) * Nt;
#pragma unroll
      for (int q = 0; q < PPW; ++q)
#pragma unroll
        for (int e = 0; e < EPP; ++e) M[ant(q, e)] = m[q * EPP + e];
    }
  }
  T* vout = (T*)p.O.v;
  for (int e = tid; e < K * G; e += nthr) {
    int i = e / G, gg = e % G;
    if (g0 + gg < K) vout[((size_t)b * K + i) * K + g0 + gg] = Qs[e];
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

// slots per row = warps overlapping it: at most the pieces a row can touch
inline int bal_slots(const kz_problem& P) {
  int pieces = (P.max_support + bal::PS - 2) / bal::PS + 1;
  int W = P.n_antennas / 32;
  return pieces < W ? pieces : W;
}

inline size_t bal_smem_bytes(const kz_problem& P, int* S_out, int* hcap_out) {
  const int K = P.n_users;
  const int pieces = (P.max_support + bal::PS - 2) / bal::PS + 1;
  const int S = bal_slots(P);
  const int hcap = K * pieces * bal::PS;
  *S_out = S;
  *hcap_out = hcap;
  return bal::plan(K, P.n_antennas, S, hcap).total;
}

template <int SCH>
inline int bal_launch(const kz_problem& P, const kz_rng& R, const kz_out& O, int T_iters, char* ws, int32_t* tstop,
                      size_t smem, int S, int hcap, cudaStream_t s) {
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
  const int groups = (P.n_users + bal::G - 1) / bal::G;
  if (cudaFuncSetAttribute(kz_balanced_kernel<SCH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return -1;
  kz_balanced_kernel<SCH><<<P.n_systems * groups, P.n_antennas, smem, s>>>(a);
  kz_lockstep_finalize<<<(P.n_systems + 127) / 128, 128, 0, s>>>(tstop, groups, P.n_systems, O.n_outer,
                                                                  O.sys_converged);
  return 1;
}

inline int bal_dispatch(const kz_problem& P, int scheme, const kz_rng& R, const kz_out& O, int T_iters, char* ws,
                        int32_t* tstop, size_t smem, int S, int hcap, cudaStream_t s) {
  switch (scheme) {
    case KZ_URK: return bal_launch<KZ_URK>(P, R, O, T_iters, ws, tstop, smem, S, hcap, s);
    case KZ_SWOR_ERK: return bal_launch<KZ_SWOR_ERK>(P, R, O, T_iters, ws, tstop, smem, S, hcap, s);
    case KZ_GK: return bal_launch<KZ_GK>(P, R, O, T_iters, ws, tstop, smem, S, hcap, s);
    case KZ_GRK: return bal_launch<KZ_GRK>(P, R, O, T_iters, ws, tstop, smem, S, hcap, s);
    case KZ_VR_OGRK: return bal_launch<KZ_VR_OGRK>(P, R, O, T_iters, ws, tstop, smem, S, hcap, s);
    case KZ_AHK: return bal_launch<KZ_AHK>(P, R, O, T_iters, ws, tstop, smem, S, hcap, s);
    case KZ_VR_OAHK: return bal_launch<KZ_VR_OAHK>(P, R, O, T_iters, ws, tstop, smem, S, hcap, s);
  }
  return 0;
}

}  // namespace kz
