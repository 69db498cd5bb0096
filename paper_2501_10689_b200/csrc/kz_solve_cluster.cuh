// Cluster kernel for large arrays (complex64): gk, grk, vr-ogrk, ahk, vr-oahk over contiguous VRs, fixed T
// (LOCKSTEP, epsilon = 0) or a per-rhs residual tolerance (RESIDUAL, solve / solve_all semantics).
//
// One thread-block cluster = one system x G right-hand sides (G = 32 or 16).  CTA c of the cluster owns W
// 32-antenna chunks in two blocks spread over the array (block j at chunk (j CL + c) W/2: every CTA samples
// the whole array, so the VR coverage ramps at the edges do not unbalance the cluster) and keeps in shared
// memory only the pieces of the rows that touch its chunks, zero padded to whole chunks.  The iterate of its
// rhs stays in registers: G = 32: lane (a, g), a = lane >> 4, holds rhs g and g + 16 on 16 antennas of its
// warp's chunk (the wide kernel's mapping); G = 16: a = lane >> 3, rhs g and g + 8 on 8 antennas.  Each h
// element loaded feeds two rhs (the SMEM/FFMA balance of csrc/kz_solve_wide.cuh).
// Rows are owned in contiguous blocks of KO = ceil(K / CL): the owner keeps q_i and r_i.
//
// Per iteration (grk; the other schemes follow the same pattern):
//   refresh  every CTA: each (row, chunk) partial goes straight into the owner's inbox IN[row][chunk slot][rhs]
//            (local store or DSMEM st.shared::cluster, drained while the next pieces compute)  -- cluster barrier
//   finalise owner: r_i = e - sum_slots IN - xi q_i (chunk order), block sums of |r_i|^2 pushed to every CTA
//                                                                                            -- cluster barrier
//   select   every CTA: the same prefix over the block sums -> the block holding the draw; its owner picks the
//            row, updates q_i, pushes (row, gamma) to every CTA                              -- cluster barrier
//   project  every CTA: m += gamma h on its chunks.
// Residual mode fuses the convergence test into the next refresh: ||r_true||^2 of the state after step t is
// the sum of the block sums of step t + 1 (grk / gk / ahk), so the stopping rule costs no extra pass; vr-oahk
// refreshes all rows (instead of its orthogonal group) at the start of each iteration for the same purpose.
// Semantics: InstanceRun.step (solvers.py:382-421), solve / StoppingRule (solvers.py:426-507).
#pragma once

#include <cstdio>
#include <cstdlib>

#include "kz_common.cuh"
#include "kz_tma.cuh"
#include "kz_solve_generic.cuh"

// timing build: close a phase before each cluster barrier so the barrier wait is its own phase
#ifdef KZ_TIMING
#define KZ_CLU_SPLIT() do { __syncthreads(); KZ_PHASE(); } while (0)
#else
#define KZ_CLU_SPLIT() do {} while (0)
#endif

namespace kz {

namespace clu {

constexpr int CH = 32;  // antennas per warp

// [owned row][rhs] arrays are XOR-swizzled so lanes-over-rows and lanes-over-rhs are both conflict free
template <int G> __device__ __forceinline__ int xo(int il, int gg) { return il * G + (gg ^ (il & 15)); }

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_ctas() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t remote(const void* p, int rank) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_remote(float2* p, int rank, float2 v) {
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(remote(p, rank)), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void st_remote(float* p, int rank, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(remote(p, rank)), "f"(v) : "memory");
}
__device__ __forceinline__ void st_remote(int* p, int rank, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(remote(p, rank)), "r"(v) : "memory");
}
__device__ __forceinline__ void st_remote(float4* p, int rank, float4 v) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(remote(p, rank)), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_cluster(uint32_t addr, float2 v) {  // addr from remote() (any CTA, own included)
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ int ld_remote(const int* p, int rank) {
  int v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(remote(p, rank)) : "memory");
  return v;
}
__device__ __forceinline__ float2 ld_remote(const float2* p, int rank) {
  float2 v;
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(remote(p, rank)) : "memory");
  return v;
}

struct Plan {
  int K, W, CL, KO, NS, pcap, nlcap;
  size_t rowS, rowL, rvo, c0, c1, en, ien, inset, loc, cost, cmask, lrow, lh, lcc, lptr, lst, optr, olst, nptr, nlst, H, Qo,
      Ro, Fo, IN, Phl, dloc, dlst, dcnt, blk, AG4, GAMv, stepv, BS, BI, SPP, NZP, DY, Dp, SEL, GAM, done, sdone, live, iters, prev, noop, conv, nchk, flops,
      misc, mbar, sptr, setn, setc, setspan, rhsv, nck, total;
};

__host__ __device__ inline size_t al(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline Plan plan(int scheme, int K, int W, int CL, int NS, int pcap, int G, int rcap,
                                      bool streamed = false) {
  Plan p;
  p.K = K;
  p.W = W;
  p.CL = CL;
  p.KO = (K + CL - 1) / CL;
  p.NS = NS;
  p.pcap = pcap;
  p.nlcap = K < pcap ? K : pcap;
  if (rcap > 0 && rcap < p.nlcap) p.nlcap = rcap;
  const int KW = (K + 31) / 32;
  const bool ogrk = scheme == KZ_VR_OGRK, oahk = scheme == KZ_VR_OAHK, gog = scheme == KZ_VR_OAHK_G;
  const bool agg = scheme == KZ_AHK || oahk || gog, greedy = !agg;  // arrays only one family touches are sized 0
  size_t o = 0;
  p.rowS = o; o = al(o + 4 * K);
  p.rowL = o; o = al(o + 4 * K);
  p.rvo = o; o = al(o + 8 * (size_t)K);
  p.c0 = o; o = al(o + 4 * K);
  p.c1 = o; o = al(o + 4 * K);
  p.en = o; o = al(o + 4 * K);
  p.ien = o; o = al(o + 4 * K);
  p.inset = o; o = al(o + K);
  p.loc = o; o = al(o + 4 * K);
  p.cost = o; o = al(o + (ogrk ? 8 * K : 0));
  p.cmask = o; o = al(o + (ogrk ? 4 * (size_t)p.KO * KW : 0));
  p.lrow = o; o = al(o + 4 * p.nlcap);
  p.lh = o; o = al(o + 4 * p.nlcap);
  p.lcc = o; o = al(o + 4 * p.nlcap);
  p.lptr = o; o = al(o + 4 * (W + 1));
  p.lst = o; o = al(o + 8 * (size_t)pcap);
  p.optr = o; o = al(o + (oahk ? 4 * (W + 1) : 0));
  p.nptr = o; o = al(o + (oahk ? 4 * (W + 1) : 0));
  p.olst = o; o = al(o + (oahk ? 8 * (size_t)pcap : 0));  // O entries then N entries (disjoint rows)
  p.nlst = p.olst;
  // one spare 16-byte unit per local row: row n starts at bank group n mod 8, so the rows a quarter-warp's
  // LDS.128 gathers in the greedy projection (one row per rhs lane) spread over the eight groups instead of
  // sharing one (chunk-padded rows alone are multiples of 256 bytes).  streamed: H from the padded global copy
  p.H = o; o = al(o + (streamed ? 0 : 8 * ((size_t)pcap * CH + 2 * (size_t)p.nlcap)));
  p.Qo = o; o = al(o + 8 * (size_t)p.KO * G);
  p.Ro = o; o = al(o + (greedy ? 8 * (size_t)p.KO * G : 0));
  p.Fo = o; o = al(o + (agg ? 8 * (size_t)p.KO * G : 0));
  p.IN = o; o = al(o + 8 * (size_t)p.KO * NS * G);
  p.Phl = o; o = al(o + (agg ? 8 * (size_t)p.nlcap * G : 0));
  p.dloc = o; o = al(o + 4 * (size_t)p.KO * CL);
  p.dlst = o; o = al(o + 4 * (size_t)p.KO * CL);
  p.dcnt = o; o = al(o + 4 * (size_t)p.KO);
  p.blk = o; o = al(o + 8 * (size_t)((K + 31) / 32));  // setup: per 32-row block (local rows, pieces)
  p.AG4 = o; o = al(o + (agg ? 16 * (size_t)CL * G : 0));
  p.GAMv = o; o = al(o + 8 * G);
  p.stepv = o; o = al(o + 4 * G);
  p.BS = o; o = al(o + 4 * (size_t)CL * G);
  p.BI = o; o = al(o + (scheme == KZ_GK ? 4 * (size_t)CL * G : 0));
  p.SPP = o; o = al(o + (greedy ? 4 * (size_t)CL * G : 0));
  p.NZP = o; o = al(o + (agg ? 4 * (size_t)CL * G : 0));
  p.DY = o; o = al(o + (agg ? 4 * (size_t)CL * G : 0));
  p.Dp = o; o = al(o + (agg ? 4 * (size_t)W * G : 0));
  p.SEL = o; o = al(o + 4 * G);
  p.GAM = o; o = al(o + 8 * G);
  p.done = o; o = al(o + 4 * G);
  p.sdone = o; o = al(o + 4 * G);
  p.live = o; o = al(o + 4 * G);
  p.iters = o; o = al(o + 4 * G);
  p.prev = o; o = al(o + 4 * G);
  p.noop = o; o = al(o + 4 * G);
  p.conv = o; o = al(o + 4 * G);
  p.nchk = o; o = al(o + 4 * G);
  p.flops = o; o = al(o + 8 * G);
  p.misc = o; o = al(o + 64);
  p.mbar = o; o = al(o + 8);
  // grouped vr-oahk: per-warp list offsets of every row set (orthogonal groups, then aggregation blocks; at most K
  // sets) and per-set row count, sum of 8 |Gamma_i| and support union (flop charges)
  p.sptr = o; o = al(o + (gog ? 4 * (size_t)W * (K + 1) : 0));
  p.setn = o; o = al(o + (gog ? 4 * (size_t)K : 0));
  p.setc = o; o = al(o + (gog ? 8 * (size_t)K : 0));
  p.setspan = o; o = al(o + (gog ? 4 * (size_t)K : 0));
  p.rhsv = o; o = al(o + 4 * (size_t)G);  // rhs of each slot (residual-mode greedy runs: grouped by |X_c|)
  p.nck = o; o = al(o + (greedy ? 4 * (size_t)K : 0));
  p.total = o;
  return p;
}

}  // namespace clu

struct CluArgs {
  kz_problem P;
  int bulk;  // stage the row pieces with bulk copies where the parity allows (kz_tma.cuh)
  kz_rng R;
  kz_out O;
  int mode;     // KZ_STOP_LOCKSTEP (fixed T) or KZ_STOP_RESIDUAL
  int cap;      // T (lockstep) or the per-rhs iteration cap
  int every;    // check_every
  float eps;    // residual tolerance
  int NS;       // inbox slots per row (= CL: any CTA may hold a piece of a row)
  int nblk;     // chunk blocks per CTA (block-interleaved slices)
  int pcap;     // (row, chunk) pairs reserved per CTA
  int rcap;     // local rows reserved per CTA (0: min(K, pcap))
  int32_t* tstop;
  const float2* hpad;  // streamed variant: H_eff padded to whole chunks, row r of system b at (b K + r) NS CH
  int order;  // residual-mode greedy runs: slots take the rhs in ascending order of their coupled-set size
};

// prepares CluArgs::hpad for the streamed variant: row r's chunk pieces c0_r .. c0_r + NS - 1, zero outside the
// support (one warp per row; coalesced 256-byte pieces)
__global__ void __launch_bounds__(256) kz_hpad_kernel(const kz_problem P, int NS, float2* hpad) {
  const long long r = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= (long long)P.n_systems * P.n_users) return;
  const int sg = P.row_seg_ptr[r];
  const int s = P.seg_start[sg], L = P.seg_len[sg];
  const int c0 = s / 32;
  const float2* src = (const float2*)P.heff + P.row_val_ptr[r];
  float2* dst = hpad + r * NS * 32;
  for (int pc = 0; pc < NS; ++pc) {
    const int ant = (c0 + pc) * 32 + lane;
    dst[pc * 32 + lane] = (ant >= s && ant < s + L) ? src[ant - s] : make_float2(0.f, 0.f);
  }
}

// GG = rhs per cluster: 16 (lane (a, g), a = lane >> 3: rhs g, g + 8 on 8 antennas) or 32 (a = lane >> 4:
// rhs g, g + 16 on 16 antennas, the wide kernel's mapping: twice the FMAs per loaded element set and per
// piece overhead, when the larger inbox fits)
// ST (streamed): H_eff is read from the padded global copy CluArgs::hpad through L1 / L2 instead of being staged
// into shared memory, so two CTAs (of different clusters) share an SM: one cluster's barrier waits and latency-bound
// phases overlap the other's FMA-bound refresh
template <int SCH, int GG, bool ST = false>
__global__ void __launch_bounds__(256, ST ? 2 : 1) kz_cluster_kernel(const __grid_constant__ CluArgs p) {
  using namespace clu;
  constexpr int G = GG;
  constexpr int NA = G == 16 ? 4 : 2;  // a-lanes sharing a (row, chunk) piece
  constexpr int LPA = 32 / NA;         // lanes per a-lane group = rhs offset of the second rhs
  constexpr int E = CH / NA;           // antennas per thread per chunk
  auto xo = [](int il, int gg) { return clu::xo<G>(il, gg); };
  using T = float2;
  constexpr bool AGG = SCH == KZ_AHK || SCH == KZ_VR_OAHK || SCH == KZ_VR_OAHK_G;
  constexpr bool GREEDY = SCH == KZ_GK || SCH == KZ_GRK || SCH == KZ_VR_OGRK;
  constexpr bool GRP = SCH == KZ_VR_OAHK_G;  // grouped vr-oahk (oracle/grouped.py): row sets in order

  extern __shared__ __align__(128) unsigned char sm[];
  const int K = p.P.n_users, Nt = p.P.n_antennas;
  const int CL = (int)cluster_ctas(), c = (int)cta_rank();
  const int ngroups = (K + G - 1) / G;
  const int cid = blockIdx.x / CL;
  const int b = cid / ngroups, grp = cid % ngroups, g0 = grp * G;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31, nthr = blockDim.x;
  const int W = nthr >> 5;
  const Plan pl = plan(SCH, K, W, CL, p.NS, p.pcap, G, p.rcap, ST);
  const int KO = pl.KO, NS = pl.NS, KW = (K + 31) / 32;
  // block-interleaved slices: CTA c owns nblk blocks of Bc = W / nblk chunks, block j at chunk
  // (j CL + c) Bc, so every CTA samples the whole array and the VR-coverage ramps at the array edges no
  // longer leave some CTAs with a fraction of the others' rows (the cluster barriers wait for the max)
  const int nblk = p.nblk, Bc = W / nblk;
  auto chunk_of = [&](int ww) { return ((ww / Bc) * CL + c) * Bc + (ww % Bc); };
  const int nch = Nt / CH;
  const int o_lo = c * KO, nown = max(0, min(K, o_lo + KO) - o_lo);
  const bool residual = p.mode == KZ_STOP_RESIDUAL;

  int* rowS = (int*)(sm + pl.rowS);
  int* rowL = (int*)(sm + pl.rowL);
  long long* rvo = (long long*)(sm + pl.rvo);  // heff offset of row i (row_val_ptr)
  int* c0 = (int*)(sm + pl.c0);
  int* c1 = (int*)(sm + pl.c1);
  float* en = (float*)(sm + pl.en);
  float* ien = (float*)(sm + pl.ien);  // 1 / e_i: aggregation / block-step weights by multiplication
  uint8_t* inset = (uint8_t*)(sm + pl.inset);
  int* loc = (int*)(sm + pl.loc);
  long long* cost = (long long*)(sm + pl.cost);
  uint32_t* cmask = (uint32_t*)(sm + pl.cmask);
  int* lrow = (int*)(sm + pl.lrow);
  int* lh = (int*)(sm + pl.lh);    // H element offset of local row n's first chunk
  int* lcc = (int*)(sm + pl.lcc);  // local chunk range of row n: lc0 | lc1 << 8
  int* lptr = (int*)(sm + pl.lptr);
  // piece lists: x = H element offset of the (row, chunk) piece | local row << 20,
  //              y = inbox offset (row, chunk slot) in the owner | (row & 15) << 20 | owner << 24
  int2* lst = (int2*)(sm + pl.lst);
  int* optr = (int*)(sm + pl.optr);
  int2* olst = (int2*)(sm + pl.olst);
  int* nptr = (int*)(sm + pl.nptr);
  int2* nlst = (int2*)(sm + pl.nlst);
  T* Hs = (T*)(sm + pl.H);
  T* Qo = (T*)(sm + pl.Qo);
  T* Ro = (T*)(sm + pl.Ro);
  T* Fo = (T*)(sm + pl.Fo);  // owned phi (aggregation weights) or gamma (orthogonal block)
  T* INs = (T*)(sm + pl.IN);
  T* Phl = (T*)(sm + pl.Phl);  // phi / gamma of the local rows, pushed by their owners
  int* dloc = (int*)(sm + pl.dloc);  // [owned row][CTA] -> local row index of the row in that CTA (-1: none)
  // (inbox: IN[owned row][chunk slot][rhs], slot = chunk - first chunk of the row, NS = max chunks per row)
  // [owned row][k] -> cluster shared address of Phl[local row] in the k-th CTA holding pieces of the row
  // (ascending CTAs; the phi push is one precomputed address per destination)
  uint32_t* dlst = (uint32_t*)(sm + pl.dlst);
  int* dcnt = (int*)(sm + pl.dcnt);
  int* blk = (int*)(sm + pl.blk);
  float4* AG4 = (float4*)(sm + pl.AG4);
  T* GAMv = (T*)(sm + pl.GAMv);
  int* stepv = (int*)(sm + pl.stepv);
  float* BS = (float*)(sm + pl.BS);
  int* BI = (int*)(sm + pl.BI);
  float* SPP = (float*)(sm + pl.SPP);
  int* NZP = (int*)(sm + pl.NZP);
  float* DY = (float*)(sm + pl.DY);
  float* Dp = (float*)(sm + pl.Dp);
  int* SEL = (int*)(sm + pl.SEL);
  T* GAM = (T*)(sm + pl.GAM);
  int* donev = (int*)(sm + pl.done);
  int* sdone = (int*)(sm + pl.sdone);  // scheme termination (InstanceRun.done)
  int* livev = (int*)(sm + pl.live);
  int* itv = (int*)(sm + pl.iters);
  int* prevv = (int*)(sm + pl.prev);
  int* noopv = (int*)(sm + pl.noop);
  int* convv = (int*)(sm + pl.conv);
  int* nchk = (int*)(sm + pl.nchk);
  long long* flv = (long long*)(sm + pl.flops);
  int* misc = (int*)(sm + pl.misc);
  int* rhsv = (int*)(sm + pl.rhsv);  // the rhs (column of V) each slot gg serves; >= K: none

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
    rvo[i] = p.P.row_val_ptr[r];
    c0[i] = s / CH;
    c1[i] = (s + L - 1) / CH;
    en[i] = (float)p.P.row_energy[r];
    ien[i] = (float)(1.0 / p.P.row_energy[r]);
    inset[i] = 0;
  }
  // slot -> rhs.  Residual-mode greedy runs: the cluster's G slots take consecutive ranks of a stable ascending sort
  // of the rhs by coupled-set size |X_c|, which tracks the iteration count to the tolerance (correlation 0.95 at
  // cfg4, tools/rhs_grouping_probe.py), so a cluster's rhs finish close together (less lockstep waste); every rhs's
  // arithmetic is unchanged (results bitwise equal to the index order)
  if (GREEDY && p.order && residual && p.P.coupled_ptr) {
    int* nck = (int*)(sm + pl.nck);
    for (int c = tid; c < K; c += nthr)
      nck[c] = p.P.coupled_ptr[(size_t)b * K + c + 1] - p.P.coupled_ptr[(size_t)b * K + c];
    for (int gg = tid; gg < G; gg += nthr) rhsv[gg] = K;
    __syncthreads();
    for (int c = tid; c < K; c += nthr) {
      const int nc = nck[c];
      int rank = 0;
      for (int j = 0; j < K; ++j) {
        const int nj = nck[j];
        rank += (nj < nc || (nj == nc && j < c)) ? 1 : 0;
      }
      if (rank >= g0 && rank < g0 + G) rhsv[rank - g0] = c;
    }
  } else {
    for (int gg = tid; gg < G; gg += nthr) rhsv[gg] = g0 + gg < K ? g0 + gg : K;
  }
  if (AGG && p.P.orth_ptr && tid == 0) {  // partition ranges read alongside the rows (one latency round)
    if (GRP) {
      misc[12] = p.P.ogrp_sys[b];
      misc[13] = p.P.ogrp_sys[b + 1];
    }
    misc[8] = p.P.orth_ptr[b];
    misc[9] = p.P.orth_ptr[b + 1];
    misc[10] = p.P.non_ptr[b];
    misc[11] = p.P.non_ptr[b + 1];
  }
  __syncthreads();
  KZ_SETUP_MARK(0);
  if (GRP) {  // set ids: 1 + group index for the orthogonal groups, then one per block of agg_cap N rows
    const int g0s = misc[12], ngs = misc[13] - misc[12], cap = p.P.agg_cap > 0 ? p.P.agg_cap : K;
    for (int gi = 0; gi < ngs; ++gi)
      for (int q = p.P.ogrp_ptr[g0s + gi] + tid; q < p.P.ogrp_ptr[g0s + gi + 1]; q += nthr)
        inset[p.P.orth_idx[q]] = (uint8_t)(1 + gi);
    for (int q = misc[10] + tid; q < misc[11]; q += nthr) inset[p.P.non_idx[q]] = (uint8_t)(1 + ngs + (q - misc[10]) / cap);
    if (tid == 0) misc[14] = ngs + (misc[11] - misc[10] + cap - 1) / cap;
  } else if (AGG && p.P.orth_ptr) {
    for (int q = misc[8] + tid; q < misc[9]; q += nthr) inset[p.P.orth_idx[q]] = 1;
    for (int q = misc[10] + tid; q < misc[11]; q += nthr) inset[p.P.non_idx[q]] = 2;
  }
  // rows touching this slice, ascending: 32-row blocks spread over the warps, two ballot passes around a
  // block-level prefix (local row index and H piece offset of every row)
  const int nblk32 = (K + 31) / 32;
  auto row_span = [&](int i, int& l0, int& l1) {  // local warps whose chunks lie in [c0_i, c1_i] (contiguous)
    l0 = W;
    l1 = -1;
    if (i < K)
      for (int ww = 0; ww < W; ++ww) {
        const int ch = chunk_of(ww);
        if (ch >= c0[i] && ch <= c1[i] && ch < nch) {
          l0 = min(l0, ww);
          l1 = ww;
        }
      }
  };
  for (int bk = w; bk < nblk32; bk += W) {
    int l0, l1;
    row_span(bk * 32 + lane, l0, l1);
    const bool ov = l0 <= l1;
    int np = ov ? l1 - l0 + 1 : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) np += __shfl_xor_sync(FULL, np, o);
    const int cnt = __popc(__ballot_sync(FULL, ov));
    if (lane == 0) {
      blk[2 * bk] = cnt;
      blk[2 * bk + 1] = np;
    }
  }
  __syncthreads();
  for (int bk = w; bk < nblk32; bk += W) {
    int n = 0, hcar = 0;
    for (int q = 0; q < bk; ++q) {
      n += blk[2 * q];
      hcar += blk[2 * q + 1];
    }
    const int i = bk * 32 + lane;
    int l0, l1;
    row_span(i, l0, l1);
    const bool ov = l0 <= l1;
    const unsigned bal = __ballot_sync(FULL, ov);
    const int np = ov ? l1 - l0 + 1 : 0;
    int sc = np;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t2 = __shfl_up_sync(FULL, sc, o);
      if (lane >= o) sc += t2;
    }
    const int idx = n + __popc(bal & ((1u << lane) - 1));
    if (i < K) loc[i] = ov ? idx : -1;
    if (ov && idx < pl.nlcap) {
      lrow[idx] = i;
      lh[idx] = (hcar + sc - np) * CH + 2 * idx;
      lcc[idx] = l0 | (l1 << 8);
    }
  }
  if (tid == 0) {
    int n = 0, hcar = 0;
    for (int q = 0; q < nblk32; ++q) {
      n += blk[2 * q];
      hcar += blk[2 * q + 1];
    }
    misc[1] = n;
    misc[2] = hcar;
  }
  __syncthreads();
  KZ_SETUP_MARK(1);
  const int NL = misc[1], npairs = misc[2];
  if (npairs > p.pcap || NL > pl.nlcap) __trap();  // layout hint violated: fail loudly
  KZ_CHECK(!ST || (long long)K * NS * CH < (1 << 20), "cluster: streamed piece offsets fit 20 bits");
  // row pieces -> shared memory, zero padded to whole chunks: one warp per local row, lanes over the 32
  // antennas of each piece (coalesced 256 B), all issued as asynchronous copies (offsets from shared memory:
  // no dependent global load, no load latency per piece)
  if constexpr (!ST) {
    // bulk copies (kz_tma.cuh) for the rows whose packed offset has their first antenna's parity, one per
    // contiguous antenna run (a row's pieces in this CTA form at most nblk runs); 8-byte asynchronous copies
    // (zero-filled outside the support) for the others
    uint64_t* mbar = (uint64_t*)(sm + pl.mbar);
    const bool bulk = p.bulk != 0;
    if (bulk && tid == 0) tma::mbar_init(mbar, 1);
    __syncthreads();
    for (int n = w; n < NL; n += W) {
      const int i = lrow[n], l0 = lcc[n] & 0xFF, l1 = lcc[n] >> 8, h0 = lh[n];
      const int s = rowS[i], L = rowL[i];
      // the row's local pieces split into runs at the slice-block boundaries (multiples of Bc local chunks);
      // within a block the chunks are consecutive, so a run is one contiguous antenna range: lane j, run j
      unsigned fallback = ~0u;  // local pieces (bit pc) left to the asynchronous copies
      if (bulk) {
        bool done = true;
        const int j = l0 / Bc + lane;
        if (j <= l1 / Bc) {
          const int la = max(l0, j * Bc), lb = min(l1, j * Bc + Bc - 1);
          done = tma::stage_run_bulk(Hs + h0 + (la - l0) * CH, heff, rvo[i], s, L, chunk_of(la) * CH,
                                     (chunk_of(lb) + 1) * CH, p.P.val_lo, p.P.val_hi, mbar);
        }
        const unsigned fb = __ballot_sync(FULL, !done);  // runs that fell back
        fallback = 0;
        for (int jj = 0; jj <= l1 / Bc - l0 / Bc; ++jj)
          if ((fb >> jj) & 1u) {
            const int jb = l0 / Bc + jj, la = max(l0, jb * Bc), lb = min(l1, jb * Bc + Bc - 1);
            fallback |= ((lb - la + 1 >= 32) ? ~0u : ((1u << (lb - la + 1)) - 1u)) << (la - l0);
          }
      }
      const T* src = heff + rvo[i];
      for (int pc = 0; pc <= l1 - l0; ++pc) {
        if (!((fallback >> pc) & 1u)) continue;
        const int ant = chunk_of(l0 + pc) * CH + lane;
        const bool in = ant >= s && ant < s + L;
        cp_async8(Hs + h0 + pc * CH + lane, src + (in ? ant - s : 0), in);
      }
    }
    if (bulk) {
      __syncthreads();
      if (tid == 0) tma::mbar_arrive(mbar);
    }
    KZ_SETUP_MARK(2);
    cp_async_wait_all();
    if (bulk) {
      tma::mbar_wait(mbar, 0);
      // zero the first / last piece's antennas outside the support (a widened bulk range pulls in a neighbour)
      for (int n = w; n < NL; n += W) {
        const int i = lrow[n], l0 = lcc[n] & 0xFF, l1 = lcc[n] >> 8, h0 = lh[n];
        const int s = rowS[i], L = rowL[i];
        for (int pc = 0; pc <= l1 - l0; pc += max(1, l1 - l0)) {
          const int ant = chunk_of(l0 + pc) * CH + lane;
          if (ant < s || ant >= s + L) Hs[h0 + pc * CH + lane] = make_float2(0.f, 0.f);
        }
      }
    }
  }
  KZ_SETUP_MARK(3);
  // per-chunk piece lists (ascending rows): all rows (lst) and, for vr-oahk, the O rows then the N rows
  // (olst / nlst share one array); one counting pass and one fill pass for all of them
  const bool want_all = (SCH != KZ_VR_OAHK && !GRP) || residual;
  constexpr bool want_on = SCH == KZ_VR_OAHK;
  // H element offset of local row n's piece on local warp ww (l0: the row's first local warp)
  auto hoff_of = [&](int n, int ww, int l0) -> int {
    if constexpr (ST) {
      const int i = lrow[n];
      return (i * NS + chunk_of(ww) - c0[i]) * CH;
    }
    return lh[n] + (ww - l0) * CH;
  };
  auto entry = [&](int n, int l0) {
    const int i = lrow[n], o = i / KO, il = i - o * KO;
    const int slot = chunk_of(w) - c0[i];
    KZ_CHECK(slot >= 0 && slot < NS && o < CL, "cluster: piece slot / owner");
    return make_int2(hoff_of(n, w, l0) | (n << 20), ((il * NS + slot) * G) | ((il & 15) << 20) | (o << 24));
  };
  {
    int ca = 0, co = 0, cn = 0;
    for (int base = 0; base < NL; base += 32) {
      const int n = base + lane;
      bool ov = false;
      int set = 0;
      if (n < NL) {
        const int l0 = lcc[n] & 0xFF, l1 = lcc[n] >> 8;
        ov = l0 <= w && w <= l1;
        set = inset[lrow[n]];
      }
      ca += __popc(__ballot_sync(FULL, ov));
      co += __popc(__ballot_sync(FULL, ov && set == 1));
      cn += __popc(__ballot_sync(FULL, ov && set == 2));
    }
    if (lane == 0) {
      if (want_all) lptr[w + 1] = ca;
      if (want_on) {
        optr[w + 1] = co;
        nptr[w + 1] = cn;
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    if (want_all) {
      lptr[0] = 0;
      for (int ww = 0; ww < W; ++ww) lptr[ww + 1] += lptr[ww];
    }
    if (want_on) {
      optr[0] = 0;
      for (int ww = 0; ww < W; ++ww) optr[ww + 1] += optr[ww];
      nptr[0] = optr[W];
      for (int ww = 0; ww < W; ++ww) nptr[ww + 1] += nptr[ww];
    }
  }
  __syncthreads();
  {
    int qa = want_all ? lptr[w] : 0, qo = want_on ? optr[w] : 0, qn = want_on ? nptr[w] : 0;
    for (int base = 0; base < NL; base += 32) {
      const int n = base + lane;
      bool ov = false;
      int set = 0, l0 = 0;
      if (n < NL) {
        l0 = lcc[n] & 0xFF;
        const int l1 = lcc[n] >> 8;
        ov = l0 <= w && w <= l1;
        set = inset[lrow[n]];
      }
      const unsigned ba = __ballot_sync(FULL, ov);
      const unsigned bo = __ballot_sync(FULL, ov && set == 1);
      const unsigned bn = __ballot_sync(FULL, ov && set == 2);
      const unsigned below = (1u << lane) - 1;
      if (ov) {
        const int2 e = entry(n, l0);
        if (want_all) lst[qa + __popc(ba & below)] = e;
        if (want_on && set == 1) olst[qo + __popc(bo & below)] = e;
        if (want_on && set == 2) nlst[qn + __popc(bn & below)] = e;
      }
      qa += __popc(ba);
      qo += __popc(bo);
      qn += __popc(bn);
    }
  }
  int* sptr = (int*)(sm + pl.sptr);
  int* setn = (int*)(sm + pl.setn);
  long long* setc = (long long*)(sm + pl.setc);
  int* setspan = (int*)(sm + pl.setspan);
  const int nset = GRP ? misc[14] : 0, ngs = GRP ? misc[13] - misc[12] : 0;
  if constexpr (GRP) {
    if (nset > K || nset > 254) __trap();  // set ids are uint8 and the tables hold K sets
    // one list per warp, ordered by set (one ballot pass per set), sptr[w (K+1) + s] = start of set s + 1
    int tot = 0;
    for (int base = 0; base < NL; base += 32) {
      const int n = base + lane;
      const bool ov = n < NL && (lcc[n] & 0xFF) <= w && w <= (lcc[n] >> 8);
      tot += __popc(__ballot_sync(FULL, ov));
    }
    if (lane == 0) lptr[w + 1] = tot;
    __syncthreads();
    if (tid == 0) {
      lptr[0] = 0;
      for (int ww = 0; ww < W; ++ww) lptr[ww + 1] += lptr[ww];
    }
    __syncthreads();
    int q = lptr[w];
    for (int st = 1; st <= nset; ++st) {
      if (lane == 0) sptr[w * (K + 1) + st - 1] = q;
      for (int base = 0; base < NL; base += 32) {
        const int n = base + lane;
        const int l0 = n < NL ? (lcc[n] & 0xFF) : 0;
        const bool ov = n < NL && l0 <= w && w <= (lcc[n] >> 8) && inset[lrow[n]] == st;
        const unsigned bal = __ballot_sync(FULL, ov);
        if (ov) lst[q + __popc(bal & ((1u << lane) - 1))] = entry(n, l0);
        q += __popc(bal);
      }
    }
    if (lane == 0) sptr[w * (K + 1) + nset] = q;
    KZ_CHECK(q == lptr[w + 1], "cluster grouped: every piece in one set");
    // per set (warp per set): rows, sum of 8 |Gamma_i| and the union of the supports (coverage bitmap, lane = word)
    for (int st = w; st < nset; st += W) {
      int n = 0, cnt = 0;
      long long c8 = 0;
      for (int w0 = 0; w0 < Nt / 32; w0 += 32) {
        const int wd = w0 + lane;
        uint32_t bits = 0;
        for (int i = 0; i < K; ++i) {
          if (inset[i] != st + 1) continue;
          if (w0 == 0) {
            n += 1;
            c8 += 8LL * rowL[i];
          }
          const int lo = max(rowS[i], 32 * wd), hi = min(rowS[i] + rowL[i], 32 * wd + 32);
          if (lo < hi) bits |= (hi - lo == 32 ? ~0u : ((1u << (hi - lo)) - 1u)) << (lo - 32 * wd);
        }
        if (wd < Nt / 32) cnt += __popc(bits);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
      if (lane == 0) {
        setn[st] = n;
        setc[st] = c8;
        setspan[st] = cnt;
      }
    }
  }
  KZ_SETUP_MARK(4);
  if constexpr (SCH == KZ_VR_OGRK) {
    // owner: bitmask of X_i for its rows (coupling is symmetric: i in X_j <=> j in X_i, vrgraph.py:60-82);
    // every CTA: the refresh cost of each X_j (flop charge)
    for (int i = tid; i < K; i += nthr) {
      const size_t r = (size_t)b * K + i;
      const int il = i - o_lo;
      const bool own = il >= 0 && il < nown;
      if (own)
        for (int q = 0; q < KW; ++q) cmask[il * KW + q] = 0;
      long long cst = 0;
      for (int q = p.P.coupled_ptr[r]; q < p.P.coupled_ptr[r + 1]; ++q) {
        const int j = p.P.coupled_idx[q];
        if (own) cmask[il * KW + (j >> 5)] |= 1u << (j & 31);
        cst += 8LL * rowL[j] + 4;
      }
      cost[i] = cst;
    }
  }
  for (int e = tid; e < KO * G; e += nthr) {
    const int il = e / G, gg = e % G;
    Qo[xo(il, gg)] = make_float2(0.f, 0.f);
    Ro[xo(il, gg)] = make_float2(o_lo + il == rhsv[gg] ? 1.f : 0.f, 0.f);
    Fo[xo(il, gg)] = make_float2(0.f, 0.f);
  }
  for (int gg = tid; gg < G; gg += nthr) {
    donev[gg] = rhsv[gg] < K ? 0 : 1;
    sdone[gg] = 0;
    livev[gg] = 0;
    itv[gg] = 0;
    prevv[gg] = -1;
    noopv[gg] = 0;
    convv[gg] = 0;
    nchk[gg] = 0;
    flv[gg] = 0;
    SEL[gg] = -1;
  }
  long long costO = 0, costN = 0;
  int nN = 0;
  if constexpr (AGG) {  // lanes over rows, every warp the same fixed-order reduction
    for (int i = lane; i < K; i += 32) {
      if (inset[i] == 1) costO += 8LL * rowL[i] + 4;
      if (inset[i] == 2) { costN += 8LL * rowL[i]; ++nN; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      costO += __shfl_xor_sync(FULL, costO, o);
      costN += __shfl_xor_sync(FULL, costN, o);
      nN += __shfl_xor_sync(FULL, nN, o);
    }
  }
  const int unionN = (AGG && p.P.non_union_size) ? p.P.non_union_size[b] : 0;
  KZ_SETUP_MARK(5);
  cluster_sync();  // every CTA of the cluster is resident and initialised before any DSMEM traffic
  KZ_SETUP_MARK(6);
  for (int e = tid; e < nown * CL; e += nthr) {  // owner: where each CTA keeps its piece of an owned row
    const int il = e / CL, d = e % CL, i = o_lo + il;
    dloc[e] = d == c ? loc[i] : ld_remote(loc + i, d);
  }
  __syncthreads();
  for (int il = tid; il < nown; il += nthr) {
    int n = 0;
    for (int d = 0; d < CL; ++d)
      if (dloc[il * CL + d] >= 0) dlst[il * CL + n++] = remote(Phl + (size_t)dloc[il * CL + d] * G, d);
    dcnt[il] = n;
  }
  __syncthreads();
  KZ_SETUP_MARK(7);
  KZ_PHASE();

  const int a = lane / LPA, g = lane % LPA;
  const int hf = lane >> 4, hl = lane & 15;  // half-warp serving one rhs in the owner / selection phases
  const unsigned hmask = 0xFFFFu << (16 * hf);
  T m0[E], m1[E];  // rhs g and g + LPA
#pragma unroll
  for (int k = 0; k < E; ++k) m0[k] = m1[k] = make_float2(0.f, 0.f);
  const float4* H4 = ST ? reinterpret_cast<const float4*>(p.hpad + (size_t)b * K * NS * CH)
                        : reinterpret_cast<const float4*>(Hs);
  // streamed: read-only global loads (L1-cached, the slice's pieces are re-read every iteration)
  auto ldh = [](const float4* q) -> float4 {
    if constexpr (ST) return __ldg(q);
    return *q;
  };

  // conj(h) . m over this warp's chunk for both rhs, reduced over the a-lanes; lane < G ends with rhs lane
  const int hcap_el = ST ? K * NS * CH : pl.pcap * CH + 2 * pl.nlcap;  // elements of H_eff the kernel may read
  auto dot16 = [&](int h0) -> T {
    KZ_CHECK(h0 >= 0 && (h0 & 1) == 0 && h0 + CH <= hcap_el, "cluster: refresh piece inside H");
    const float4* hp = H4 + (h0 >> 1) + a;
    float x0 = 0.f, y0 = 0.f, x1 = 0.f, y1 = 0.f, u0 = 0.f, v0 = 0.f, u1 = 0.f, v1 = 0.f;
#pragma unroll
    for (int j = 0; j < E / 2; ++j) {
      const float4 h = ldh(hp + NA * j);
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
    const float px = x0 + x1, py = y0 + y1, qx = u0 + u1, qy = v0 + v1;
    const bool odd = a & 1;  // odd a-lanes keep rhs g + LPA
    const float sx = odd ? px : qx, sy = odd ? py : qy;
    const float rx = __shfl_xor_sync(FULL, sx, LPA), ry = __shfl_xor_sync(FULL, sy, LPA);
    float kx = (odd ? qx : px) + rx, ky = (odd ? qy : py) + ry;
    if constexpr (NA == 4) {
      kx += __shfl_xor_sync(FULL, kx, 16);
      ky += __shfl_xor_sync(FULL, ky, 16);
    }
    return make_float2(kx, ky);
  };
  // partial of each (row, chunk) piece straight into the owner's inbox (local or DSMEM store): no slice-level
  // staging, the remote stores drain while the warp computes its next pieces
  auto deliver = [&](int2 e, T v) {
    if (lane < G) {
      T* dst = INs + (e.y & 0xFFFFF) + (lane ^ ((e.y >> 20) & 15));
      const int o = e.y >> 24;
      KZ_CHECK(o < CL && (e.y & 0xFFFFF) + G <= KO * NS * G, "cluster: inbox slot (DSMEM) index");
      if (o == c) *dst = v; else st_remote(dst, o, v);
    }
  };
  auto refresh_range = [&](int q, const int q1, const int2* L) {
    for (; q + 3 < q1; q += 4) {  // four pieces in flight
      const int2 e0 = L[q], e1 = L[q + 1], e2 = L[q + 2], e3 = L[q + 3];
      const T v0 = dot16(e0.x & 0xFFFFF);
      const T v1 = dot16(e1.x & 0xFFFFF);
      const T v2 = dot16(e2.x & 0xFFFFF);
      const T v3 = dot16(e3.x & 0xFFFFF);
      deliver(e0, v0);
      deliver(e1, v1);
      deliver(e2, v2);
      deliver(e3, v3);
    }
    for (; q + 1 < q1; q += 2) {
      const int2 e0 = L[q], e1 = L[q + 1];
      const T v0 = dot16(e0.x & 0xFFFFF);
      const T v1 = dot16(e1.x & 0xFFFFF);
      deliver(e0, v0);
      deliver(e1, v1);
    }
    if (q < q1) deliver(L[q], dot16(L[q].x & 0xFFFFF));
  };
  auto refresh = [&](const int* ptr, const int2* L) { refresh_range(ptr[w], ptr[w + 1], L); };
  // owner: residual of owned row il for rhs gg from the slice sums (fixed slice order)
  auto oresid = [&](int il, int gg, bool dense) -> T {
    const int i = o_lo + il;
    const T* pp = INs + (size_t)il * NS * G + (gg ^ (il & 15));
    const int ns = c1[i] - c0[i];
    float dx = 0.f, dy = 0.f;
    for (int sl = 0; sl <= ns; ++sl) {  // the row's chunk pieces, ascending (fixed order)
      const T v = pp[sl * G];
      dx += v.x;
      dy += v.y;
    }
    const T q = Qo[xo(il, gg)];
    if (dense) {  // solvers.py:149-153
      T r = make_float2(-dx - q.x * regf, -dy - q.y * regf);
      if (i == rhsv[gg]) r.x += 1.f;
      return r;
    }
    const float tg = i == rhsv[gg] ? 1.f : 0.f;  // solvers.py:166
    return make_float2((tg - dx) - q.x * regf, (0.f - dy) - q.y * regf);
  };
  auto push_phi = [&](int il, int gg, T v) {
    const int nd = dcnt[il];
    KZ_CHECK(il >= 0 && il < KO && nd <= CL && gg < G, "cluster: phi destinations");
    const uint32_t* da = dlst + il * CL;
    const uint32_t off = 8u * (uint32_t)gg;
#pragma unroll 4
    for (int k = 0; k < nd; ++k) st_cluster(da[k] + off, v);
  };
  // owner: phi = r / e on its rows of set `which` (0 = all), pushed to the slices; block partials of
  // vdot(phi, r), ||phi||^2, ||r||^2 and any(phi != 0) pushed to every CTA (solvers.py:240-254, 274)
  auto owner_weights = [&](int which, bool gate_live) {
    for (int pair = w; pair < G / 2; pair += W) {
      const int gg = pair + hf * (G / 2);
      float nx = 0.f, ny = 0.f, sp = 0.f, n2 = 0.f;
      bool nz = false;
      if (gate_live ? livev[gg] != 0 : !donev[gg])
        for (int il = hl; il < nown; il += 16) {
          const int i = o_lo + il;
          if (which && inset[i] != which) continue;
          const T r = oresid(il, gg, which == 0);
          const float ie = ien[i];
          const T ph = make_float2(r.x * ie, r.y * ie);
          Fo[xo(il, gg)] = ph;
          push_phi(il, gg, ph);
          nz |= (ph.x != 0.f || ph.y != 0.f);
          nx = fmaf(ph.x, r.x, nx); nx = fmaf(ph.y, r.y, nx);
          ny = fmaf(ph.x, r.y, ny); ny = fmaf(-ph.y, r.x, ny);
          sp = fmaf(ph.x, ph.x, sp); sp = fmaf(ph.y, ph.y, sp);
          n2 = fmaf(r.x, r.x, fmaf(r.y, r.y, n2));
        }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {
        nx += __shfl_xor_sync(FULL, nx, o);
        ny += __shfl_xor_sync(FULL, ny, o);
        sp += __shfl_xor_sync(FULL, sp, o);
        n2 += __shfl_xor_sync(FULL, n2, o);
      }
      const int anz = (__ballot_sync(FULL, nz) & hmask) ? 1 : 0;
      if (hl < CL) {
        const int d = hl, k = c * G + gg;
        const float4 v = make_float4(nx, ny, sp, n2);
        if (d == c) {
          AG4[k] = v;
          NZP[k] = anz;
        } else {
          st_remote(AG4 + k, d, v);
          st_remote(NZP + k, d, anz);
        }
      }
    }
  };
  auto project = [&](T (&mr)[E], int n, T gm) {  // m += gm h on this warp's chunk of local row n
    const int l0 = lcc[n] & 0xFF, l1 = lcc[n] >> 8;
    if (w < l0 || w > l1) return;
    KZ_CHECK(n >= 0 && n < pl.nlcap && hoff_of(n, w, l0) + CH <= hcap_el, "cluster: projected piece inside H");
    const float4* hp = H4 + (hoff_of(n, w, l0) >> 1) + a;
#pragma unroll
    for (int j = 0; j < E / 2; ++j) {
      const float4 h = ldh(hp + NA * j);
      const int k = 2 * j;
      mr[k].x = fmaf(gm.x, h.x, mr[k].x); mr[k].x = fmaf(-gm.y, h.y, mr[k].x);
      mr[k].y = fmaf(gm.x, h.y, mr[k].y); mr[k].y = fmaf(gm.y, h.x, mr[k].y);
      mr[k + 1].x = fmaf(gm.x, h.z, mr[k + 1].x); mr[k + 1].x = fmaf(-gm.y, h.w, mr[k + 1].x);
      mr[k + 1].y = fmaf(gm.x, h.w, mr[k + 1].y); mr[k + 1].y = fmaf(gm.y, h.z, mr[k + 1].y);
    }
  };
  auto draw_u = [&](int gg) -> double {
    const int cc = rhsv[gg], d = itv[gg];
    if (p.R.kind == KZ_RNG_PHILOX) return philox_uniform(p.R.seed, (uint32_t)(b + p.R.system_base), (uint32_t)cc, (uint64_t)d);
    return p.R.uniforms[((size_t)b * K + cc) * p.R.stream_len + d];
  };
  // residual-mode stopping test of the state after step itv (solvers.py:480-503); returns true if the rhs stops
  auto stop_test = [&](int gg, float nrm2) -> bool {
    if (!residual) return false;
    const int it = itv[gg];
    if (it >= 1 && it % p.every == 0) {
      nchk[gg] += 1;
      if (sqrtf(nrm2) <= p.eps) {
        convv[gg] = 1;
        donev[gg] = 1;
        return true;
      }
    }
    if (it >= p.cap) {
      donev[gg] = 1;
      return true;
    }
    return false;
  };

  const long long dense_refresh = 6LL * K * Nt + 2LL * K * (Nt + 1) + 2LL * K;
  const long long dense_rk = 2 + 8LL * Nt + 2;
  // charge of one greedy selection pass (refresh + selection), before the step itself
  auto sel_cost = [&](int gg) -> long long {
    if (SCH == KZ_GK) return dense_refresh + 4LL * K;
    if (SCH == KZ_GRK) return dense_refresh + 4LL * K + 2;
    return (prevv[gg] >= 0 ? cost[prevv[gg]] : 0) + 4LL * K + 2;
  };
  // aggregated projection over the list entries [q0, q1) (solvers.py:257-309): y = sum_i phi_i h_i (ascending
  // rows), den = ||y||^2 + xi ||phi||^2 from fixed-order reductions over warps and CTAs, then m += gamma y and the
  // owners' q += gamma phi over their rows of set qset (0: every row); nrows / ycost / span: the ahk_step charges
  auto agg_step = [&](int q0, const int q1, const int2* L, int nrows, long long ycost, int span, int qset) {
      T y0[E], y1[E];
#pragma unroll
      for (int k = 0; k < E; ++k) y0[k] = y1[k] = make_float2(0.f, 0.f);
      int q = q0;
      for (; q + 1 < q1; q += 2) {  // two pieces in flight
        const int e0 = L[q].x, e1 = L[q + 1].x, n0 = e0 >> 20, n1 = e1 >> 20;
        KZ_CHECK(n0 < pl.nlcap && n1 < pl.nlcap && (e0 & 0xFFFFF) + CH <= hcap_el && (e1 & 0xFFFFF) + CH <= hcap_el,
                 "cluster: aggregated pieces inside H / Phl");
        const T p00 = Phl[n0 * G + g], p01 = Phl[n0 * G + g + LPA];
        const T p10 = Phl[n1 * G + g], p11 = Phl[n1 * G + g + LPA];
        const float4* hp0 = H4 + ((e0 & 0xFFFFF) >> 1) + a;
        const float4* hp1 = H4 + ((e1 & 0xFFFFF) >> 1) + a;
#pragma unroll
        for (int j = 0; j < E / 2; ++j) {
          const float4 h0 = ldh(hp0 + NA * j), h1 = ldh(hp1 + NA * j);
          const int k = 2 * j;
          y0[k] = cfma(p00, make_float2(h0.x, h0.y), y0[k]);
          y0[k + 1] = cfma(p00, make_float2(h0.z, h0.w), y0[k + 1]);
          y1[k] = cfma(p01, make_float2(h0.x, h0.y), y1[k]);
          y1[k + 1] = cfma(p01, make_float2(h0.z, h0.w), y1[k + 1]);
          y0[k] = cfma(p10, make_float2(h1.x, h1.y), y0[k]);
          y0[k + 1] = cfma(p10, make_float2(h1.z, h1.w), y0[k + 1]);
          y1[k] = cfma(p11, make_float2(h1.x, h1.y), y1[k]);
          y1[k + 1] = cfma(p11, make_float2(h1.z, h1.w), y1[k + 1]);
        }
      }
      if (q < q1) {
        const int e0 = L[q].x, n0 = e0 >> 20;
        const T p00 = Phl[n0 * G + g], p01 = Phl[n0 * G + g + LPA];
        const float4* hp0 = H4 + ((e0 & 0xFFFFF) >> 1) + a;
#pragma unroll
        for (int j = 0; j < E / 2; ++j) {
          const float4 h0 = ldh(hp0 + NA * j);
          const int k = 2 * j;
          y0[k] = cfma(p00, make_float2(h0.x, h0.y), y0[k]);
          y0[k + 1] = cfma(p00, make_float2(h0.z, h0.w), y0[k + 1]);
          y1[k] = cfma(p01, make_float2(h0.x, h0.y), y1[k]);
          y1[k + 1] = cfma(p01, make_float2(h0.z, h0.w), y1[k + 1]);
        }
      }
      float s0 = 0.f, s1 = 0.f;
#pragma unroll
      for (int k = 0; k < E; ++k) {
        s0 = fmaf(y0[k].x, y0[k].x, fmaf(y0[k].y, y0[k].y, s0));
        s1 = fmaf(y1[k].x, y1[k].x, fmaf(y1[k].y, y1[k].y, s1));
      }
#pragma unroll
      for (int o = LPA; o < 32; o <<= 1) {
        s0 += __shfl_xor_sync(FULL, s0, o);
        s1 += __shfl_xor_sync(FULL, s1, o);
      }
      if (a == 0) {
        Dp[w * G + g] = s0;
        Dp[w * G + g + LPA] = s1;
      }
      __syncthreads();
      if (tid < G) {
        float dy = 0.f;
        for (int ww = 0; ww < W; ++ww) dy += Dp[ww * G + tid];
        for (int d = 0; d < CL; ++d) {
          float* dst = DY + c * G + tid;
          if (d == c) *dst = dy; else st_remote(dst, d, dy);
        }
      }
      cluster_sync();
      KZ_PHASE();
      // step length per rhs (identical in every CTA: fixed-order sums of the pushed partials)
      if (tid < G) {
        const int gg = tid;
        bool live = livev[gg];
        if (SCH == KZ_AHK) {
          live = false;
          if (!donev[gg]) {
            float n2 = 0.f;
            for (int d = 0; d < CL; ++d) n2 += AG4[d * G + gg].w;
            if (!stop_test(gg, n2)) {
              live = true;
              flv[gg] += dense_refresh + 2LL * K;
            }
          }
          livev[gg] = live;
        }
        stepv[gg] = 0;
        if (live) {
          float nx = 0.f, ny = 0.f, sp = 0.f, den = 0.f;
          int nz = 0;
          for (int d = 0; d < CL; ++d) {
            const float4 v = AG4[d * G + gg];
            nx += v.x; ny += v.y; sp += v.z; nz |= NZP[d * G + gg];
            den += DY[d * G + gg];
          }
          den = fmaf(regf, sp, den);
          const int n = nrows;
          if (SCH != KZ_AHK) flv[gg] += 2LL * nrows;  // aggregation_weights charge
          bool step = false;
          if (nz && n > 0) {
            long long f = 6LL * n + 2LL * max(n - 1, 0) + ycost + 4LL * span + 3LL * n + 2;
            if (den != 0.f) {
              step = true;
              f += 2 + 8LL * span + 8LL * n;
              GAMv[gg] = make_float2(nx / den, ny / den);
            }
            flv[gg] += f;
          }
          if (step) {
            stepv[gg] = 1;
            if (SCH == KZ_AHK) itv[gg] += 1;
          } else {
            noopv[gg] += 1;
            if (SCH == KZ_AHK) {  // ahk_step returned False: InstanceRun.done (solvers.py:407-413)
              donev[gg] = 1;
              sdone[gg] = 1;
              if (residual) {
                nchk[gg] += 1;
                convv[gg] = 1;
              }
            }
          }
        }
      }
      __syncthreads();
      if (stepv[g]) {
        const T gm = GAMv[g];
#pragma unroll
        for (int k = 0; k < E; ++k) m0[k] = cfma(gm, y0[k], m0[k]);
      }
      if (stepv[g + LPA]) {
        const T gm = GAMv[g + LPA];
#pragma unroll
        for (int k = 0; k < E; ++k) m1[k] = cfma(gm, y1[k], m1[k]);
      }
      // owner: q += gamma phi over its aggregated rows
      for (int e = tid; e < nown * G; e += nthr) {
        const int il = e / G, gg = e % G;
        if (!stepv[gg] || (qset > 0 && inset[o_lo + il] != qset)) continue;
        Qo[xo(il, gg)] = cfma(GAMv[gg], Fo[xo(il, gg)], Qo[xo(il, gg)]);
      }
  };
  int t;
  for (t = 1;; ++t) {
    KZ_ITER();
    if constexpr (GREEDY) {
      refresh(lptr, lst);
      KZ_CLU_SPLIT();
      cluster_sync();
      KZ_PHASE();
      // owner: residuals of its rows, block sums (grk / vr-ogrk) or block argmax (gk); half-warp per rhs
      for (int pair = w; pair < G / 2; pair += W) {
        const int gg = pair + hf * (G / 2);
        const bool act = !donev[gg];
        float ws = 0.f, fresh = 0.f, best = -1.f;
        int bi = 0x7fffffff;
        if (act)
          for (int il = hl; il < nown; il += 16) {
            const int i = o_lo + il;
            bool upd = true;
            if constexpr (SCH == KZ_VR_OGRK) {
              const int pr = prevv[gg];
              upd = pr >= 0 && ((cmask[il * KW + (pr >> 5)] >> (pr & 31)) & 1u);
            }
            T r;
            if (upd || residual) {
              const T rf = oresid(il, gg, SCH != KZ_VR_OGRK);
              fresh += rf.x * rf.x + rf.y * rf.y;
              r = upd ? rf : Ro[xo(il, gg)];
            } else {
              r = Ro[xo(il, gg)];
            }
            if (upd) Ro[xo(il, gg)] = r;
            const float w2 = r.x * r.x + r.y * r.y;
            ws += w2;
            if constexpr (SCH == KZ_GK) {
              const float sc = w2 / en[i];
              if (sc > best) { best = sc; bi = i; }
            }
          }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
          ws += __shfl_xor_sync(FULL, ws, o);
          fresh += __shfl_xor_sync(FULL, fresh, o);
          if constexpr (SCH == KZ_GK) {
            const float ob = __shfl_xor_sync(FULL, best, o);
            const int oi = __shfl_xor_sync(FULL, bi, o);
            if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
          }
        }
        if (hl < CL) {
          const int d = hl;
          if (SCH == KZ_GK) {
            float* bs = BS + c * G + gg;
            int* bx = BI + c * G + gg;
            if (d == c) { *bs = best; *bx = bi; } else { st_remote(bs, d, best); st_remote(bx, d, bi); }
          } else {
            float* bs = BS + c * G + gg;
            if (d == c) *bs = ws; else st_remote(bs, d, ws);
          }
          float* fs = SPP + c * G + gg;  // fresh ||r||^2 partial (the stopping test)
          if (d == c) *fs = SCH == KZ_VR_OGRK ? fresh : ws; else st_remote(fs, d, SCH == KZ_VR_OGRK ? fresh : ws);
        }
      }
      KZ_CLU_SPLIT();
      cluster_sync();
      KZ_PHASE();
      // selection: the same block-level decision in every CTA, the owner of the chosen row does the step.
      // Control flow stays warp-uniform (the two half-warps serve different rhs): predicates, no early exits.
      for (int pair = w; pair < G / 2; pair += W) {
        const int gg = pair + hf * (G / 2);
        bool act = !donev[gg];
        // the draw is independent of the sums: issue it first (counter-based Philox / a stream read, consumed
        // only if a row is drawn)
        const double u_draw = (SCH != KZ_GK && act) ? draw_u(gg) : 0.0;
        // ||r||^2 of the state after the last step: butterfly over the CTAs' partials (same order in every CTA)
        float nrm2 = hl < CL ? SPP[hl * G + gg] : 0.f;
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) nrm2 += __shfl_xor_sync(FULL, nrm2, o);
        bool stopped = false;
        if (act && hl == 0) stopped = stop_test(gg, nrm2);
        stopped = __shfl_sync(FULL, stopped, 16 * hf);
        act = act && !stopped;
        const long long f = sel_cost(gg);
        int cstar = -1, isel = -1;
        if constexpr (SCH == KZ_GK) {
          float bb = act && hl < CL ? BS[hl * G + gg] : -1.f;
          int bx = act && hl < CL ? BI[hl * G + gg] : 0x7fffffff;
#pragma unroll
          for (int o = 8; o > 0; o >>= 1) {
            const float ob = __shfl_xor_sync(FULL, bb, o);
            const int oi = __shfl_xor_sync(FULL, bx, o);
            if (ob > bb || (ob == bb && oi < bx)) { bb = ob; bx = oi; }
          }
          if (act && bb > 0.f) {  // greedy-max: None if every score is zero (solvers.py:210-215)
            isel = bx;
            cstar = bx / KO;
          }
        } else {
          const float v = act && hl < CL ? BS[hl * G + gg] : 0.f;
          float incl = v;
#pragma unroll
          for (int o = 1; o < 16; o <<= 1) {
            const float t2 = __shfl_up_sync(FULL, incl, o, 16);
            if (hl >= o) incl += t2;
          }
          const float tot = __shfl_sync(FULL, incl, 16 * hf + 15);
          const bool draw = act && tot > 0.f;  // tot == 0: None, no draw consumed (solvers.py:235-236)
          const float tau = draw ? (float)u_draw * tot : 0.f;
          const unsigned hit = (__ballot_sync(FULL, draw && v > 0.f && incl > tau) & hmask) >> (16 * hf);
          const unsigned nzb = (__ballot_sync(FULL, draw && v > 0.f) & hmask) >> (16 * hf);
          if (draw) cstar = hit ? __ffs(hit) - 1 : 31 - __clz(nzb);
          const float excl = __shfl_sync(FULL, incl - v, 16 * hf + (cstar < 0 ? 0 : cstar));
          // the chosen block's owner scans its rows, 16 per step
          const bool mine = cstar == c;
          float carry = excl;
          int lastnz = -1;
          bool found = !mine;
          for (int base = 0; base < nown; base += 16) {
            if (__all_sync(FULL, found)) break;
            const int il = base + hl;
            float wv = 0.f;
            if (mine && il < nown) {
              const T r = Ro[xo(il, gg)];
              wv = r.x * r.x + r.y * r.y;
            }
            float sc = wv;
#pragma unroll
            for (int o = 1; o < 16; o <<= 1) {
              const float t2 = __shfl_up_sync(FULL, sc, o, 16);
              if (hl >= o) sc += t2;
            }
            const unsigned h2 = (__ballot_sync(FULL, !found && wv > 0.f && carry + sc > tau) & hmask) >> (16 * hf);
            const unsigned n2 = (__ballot_sync(FULL, wv > 0.f) & hmask) >> (16 * hf);
            if (!found && h2) {
              isel = o_lo + base + __ffs(h2) - 1;
              found = true;
            }
            if (n2) lastnz = o_lo + base + 31 - __clz(n2);
            carry += __shfl_sync(FULL, sc, 16 * hf + 15);
          }
          if (mine && !found) isel = lastnz;
        }
        if (act && cstar < 0 && hl == 0) {  // None: InstanceRun.done (solvers.py:391-396)
          donev[gg] = 1;
          sdone[gg] = 1;
          flv[gg] += f;
          if (residual) {  // the reference checks once more on done, then reports convergence
            nchk[gg] += 1;
            convv[gg] = 1;
          }
        }
        if (!(act && cstar >= 0) && hl == 0) SEL[gg] = -1;
        // owner: rk_step (solvers.py:173-188), then (row, gamma) to every CTA
        const bool step = act && cstar == c;
        T gm = make_float2(0.f, 0.f);
        if (step) {
          const T r = Ro[xo(isel - o_lo, gg)];
          const float e = en[isel];
          gm = make_float2(r.x / e, r.y / e);
        }
        __syncwarp();
        if (step && hl == 0) {
          const int il = isel - o_lo;
          const T q = Qo[xo(il, gg)];
          Qo[xo(il, gg)] = make_float2(q.x + gm.x, q.y + gm.y);
          Ro[xo(il, gg)] = make_float2(0.f, 0.f);
          const int it = itv[gg];
          if (p.O.rows && it < p.O.rows_cap) p.O.rows[((size_t)b * K + rhsv[gg]) * p.O.rows_cap + it] = isel;
        }
        if (step && hl < CL) {
          if (hl == c) {
            SEL[gg] = isel;
            GAM[gg] = gm;
          } else {
            st_remote(SEL + gg, hl, isel);
            st_remote(GAM + gg, hl, gm);
          }
        }
      }
      KZ_CLU_SPLIT();
      cluster_sync();
      KZ_PHASE();
      // bookkeeping of the steps (every CTA keeps the same per-rhs counters)
      if (tid < G) {
        const int gg = tid, i = SEL[gg];
        if (i >= 0) {
          const long long fr = SCH == KZ_VR_OGRK ? 2 + 8LL * rowL[i] + 2 : dense_rk;
          flv[gg] += sel_cost(gg) + fr;
          itv[gg] += 1;
          prevv[gg] = i;
        }
      }
      {
        const int i0 = SEL[g], i1 = SEL[g + LPA];
        if (i0 >= 0 && loc[i0] >= 0) project(m0, loc[i0], GAM[g]);
        if (i1 >= 0 && loc[i1] >= 0) project(m1, loc[i1], GAM[g + LPA]);
      }
    } else if constexpr (SCH == KZ_AHK) {
      refresh(lptr, lst);
      cluster_sync();
      KZ_PHASE();
      owner_weights(0, false);
      cluster_sync();
      KZ_PHASE();
    } else if constexpr (GRP) {  // grouped VR-OAHK (oracle/grouped.py GroupedRun.step), fixed T
      for (int gg = tid; gg < G; gg += nthr) livev[gg] = !donev[gg];
      __syncthreads();
      const int* sp = sptr + w * (K + 1);
      for (int st = 1; st <= nset; ++st) {
        refresh_range(sp[st - 1], sp[st], lst);
        cluster_sync();
        if (st <= ngs) {  // orthogonal group: exact block projection (solvers.py:312-332)
          for (int pair = w; pair < G / 2; pair += W) {
            const int gg = pair + hf * (G / 2);
            if (livev[gg])
              for (int il = hl; il < nown; il += 16) {
                const int i = o_lo + il;
                if (inset[i] != st) continue;
                const T r = oresid(il, gg, false);
                const T gm = make_float2(r.x * ien[i], r.y * ien[i]);
                Fo[xo(il, gg)] = gm;
                push_phi(il, gg, gm);
              }
          }
          cluster_sync();
          for (int e = tid; e < nown * G; e += nthr) {
            const int il = e / G, gg = e % G;
            if (inset[o_lo + il] != st || !livev[gg]) continue;
            const T gm = Fo[xo(il, gg)], q = Qo[xo(il, gg)];
            Qo[xo(il, gg)] = make_float2(q.x + gm.x, q.y + gm.y);
          }
          const bool l0v = livev[g], l1v = livev[g + LPA];
          for (int q = sp[st - 1]; q < sp[st]; ++q) {
            const int n = lst[q].x >> 20;
            if (l0v) project(m0, n, Phl[n * G + g]);
            if (l1v) project(m1, n, Phl[n * G + g + LPA]);
          }
          if (tid < G && livev[tid]) flv[tid] += 2 * (setc[st - 1] + 4LL * setn[st - 1]);
        } else {  // block of <= agg_cap rows: refresh, weights, aggregated step (solvers.py:417-421, 248-309)
          if (tid < G && livev[tid]) flv[tid] += setc[st - 1] + 4LL * setn[st - 1];
          owner_weights(st, true);
          cluster_sync();
          agg_step(sp[st - 1], sp[st], lst, setn[st - 1], setc[st - 1], setspan[st - 1], st);
        }
        __syncthreads();
      }
      if (tid < G && livev[tid]) itv[tid] += 1;
    } else {  // VR-OAHK (solvers.py:414-421)
      // orthogonal group O: exact block projection (solvers.py:312-332); residual mode refreshes every row
      if (residual) refresh(lptr, lst); else refresh(optr, olst);
      cluster_sync();
      KZ_PHASE();
      for (int pair = w; pair < G / 2; pair += W) {
        const int gg = pair + hf * (G / 2);
        float n2 = 0.f;
        if (!donev[gg])
          for (int il = hl; il < nown; il += 16) {
            const int i = o_lo + il;
            if (!residual && inset[i] != 1) continue;
            const T r = oresid(il, gg, false);
            if (inset[i] == 1) {
              const T gm = make_float2(r.x * ien[i], r.y * ien[i]);
              Fo[xo(il, gg)] = gm;
              push_phi(il, gg, gm);
            }
            n2 = fmaf(r.x, r.x, fmaf(r.y, r.y, n2));
          }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) n2 += __shfl_xor_sync(FULL, n2, o);
        if (residual && hl < CL) {
          const int k = c * G + gg;
          if (hl == c) BS[k] = n2; else st_remote(BS + k, hl, n2);
        }
      }
      cluster_sync();
      KZ_PHASE();
      if (tid < G) {
        const int gg = tid;
        livev[gg] = 0;
        if (!donev[gg]) {
          float n2 = 0.f;
          for (int d = 0; d < CL; ++d) n2 += BS[d * G + gg];
          if (!stop_test(gg, n2)) {
            livev[gg] = 1;
            itv[gg] += 1;
            flv[gg] += 2 * costO + (nN ? costN + 4LL * nN : 0);
          }
        }
      }
      __syncthreads();
      // owner: q_i += gamma_i on O; every CTA: m += gamma_i h_i for its O pieces (disjoint supports)
      for (int e = tid; e < nown * G; e += nthr) {
        const int il = e / G, gg = e % G;
        if (inset[o_lo + il] != 1 || !livev[gg]) continue;
        const T gm = Fo[xo(il, gg)], q = Qo[xo(il, gg)];
        Qo[xo(il, gg)] = make_float2(q.x + gm.x, q.y + gm.y);
      }
      {
        const bool l0v = livev[g], l1v = livev[g + LPA];
        for (int q = optr[w]; q < optr[w + 1]; ++q) {
          const int n = olst[q].x >> 20;
          if (l0v) project(m0, n, Phl[n * G + g]);
          if (l1v) project(m1, n, Phl[n * G + g + LPA]);
        }
      }
      KZ_PHASE();
      if (nN > 0) {
        refresh(nptr, nlst);
        cluster_sync();
        KZ_PHASE();
        owner_weights(2, true);
        cluster_sync();
        KZ_PHASE();
      }
    }
    if constexpr (AGG && SCH != KZ_VR_OAHK_G) {
      if (SCH == KZ_AHK)
        agg_step(lptr[w], lptr[w + 1], lst, K, 6LL * Nt * K + 2LL * Nt * max(K - 1, 0), Nt, 0);
      else if (nN > 0)
        agg_step(nptr[w], nptr[w + 1], nlst, nN, costN, unionN, 2);
    }
    __syncthreads();
    KZ_PHASE();
    if (!residual && t >= p.cap) break;
    bool all_done = true;
    for (int gg = 0; gg < G; ++gg)
      if (!donev[gg]) all_done = false;
    if (all_done) break;
  }
  const int t_end = t > p.cap ? p.cap : t;
  cluster_sync();  // no CTA leaves while its shared memory may still be addressed by the cluster

  // ------------------------------------------------------------------ outputs
  if (c == 0 && tid == 0 && p.tstop) p.tstop[cid] = t_end;
  if (blockIdx.x < (unsigned)p.P.n_systems * K)
    KZ_TDUMP((long long*)((char*)p.tstop + ((size_t)p.P.n_systems * p.P.n_users * 4 + 7) / 8 * 8));
  if (p.O.iterates) {
    auto store_m = [&](const T (&mr)[E], int r) {
      const int cc = rhsv[g + LPA * r], chunk = chunk_of(w);
      if (cc >= K || chunk >= Nt / CH) return;
      T* M = (T*)p.O.iterates + ((size_t)b * K + cc) * Nt + chunk * CH;
#pragma unroll
      for (int k = 0; k < E; ++k) M[2 * NA * (k >> 1) + 2 * a + (k & 1)] = mr[k];
    };
    store_m(m0, 0);
    store_m(m1, 1);
  }
  T* vout = (T*)p.O.v;
  for (int e = tid; e < nown * G; e += nthr) {
    const int il = e / G, gg = e % G;
    if (rhsv[gg] < K) vout[((size_t)b * K + o_lo + il) * K + rhsv[gg]] = Qo[xo(il, gg)];
  }
  if (c == 0)
    for (int gg = tid; gg < G; gg += nthr) {
      const int cc = rhsv[gg];
      if (cc >= K) continue;
      const size_t r = (size_t)b * K + cc;
      if (p.O.iters) p.O.iters[r] = itv[gg];
      if (p.O.converged) p.O.converged[r] = residual && convv[gg] ? 1 : 0;
      if (p.O.done) p.O.done[r] = sdone[gg] ? 1 : 0;
      if (p.O.noop_steps) p.O.noop_steps[r] = noopv[gg];
      if (p.O.flops) p.O.flops[r] = flv[gg];
      if (p.O.n_checks) p.O.n_checks[r] = nchk[gg];
    }
}

// ------------------------------------------------------------------ host side
inline size_t cluster_smem_bytes(const kz_problem& P, int scheme, int W, int G, int* CL, int* NS, int* pcap,
                                 int* rcap, bool streamed = false) {
  const int nch = P.n_antennas / clu::CH;
  *CL = (nch + W - 1) / W;
  *NS = (P.max_support + clu::CH - 2) / clu::CH + 1;  // inbox slots: chunks a row can touch
  *pcap = W == 4 ? P.slice_pairs_128 : (W == 8 ? P.slice_pairs_256 : 0);
  *rcap = W == 4 ? P.slice_rows_128 : (W == 8 ? P.slice_rows_256 : 0);
  if (*pcap <= 0) return ~size_t(0);
  return clu::plan(scheme, P.n_users, W, *CL, *NS, *pcap, G, *rcap, streamed).total;
}

// bytes of the streamed variant's padded H_eff copy (CluArgs::hpad), placed after the tstop block of the workspace
inline size_t cluster_hpad_offset(const kz_problem& P) { return kz_align(ls_extra_ws(P)); }
inline size_t cluster_hpad_bytes(const kz_problem& P, int NS) {
  return (size_t)P.n_systems * P.n_users * NS * clu::CH * sizeof(float2);
}
inline thread_local size_t g_cluster_dry_ws = 0;  // workspace the dispatched cluster variant needs (dry launches)

template <int SCH, int GG, bool ST>
inline int cluster_launch(const CluArgs& a, int W, int CL, size_t smem, cudaStream_t s) {
  auto kern = kz_cluster_kernel<SCH, GG, ST>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return -1;
  if (CL > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  const int groups = (a.P.n_users + GG - 1) / GG;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a.P.n_systems * groups * CL));
  cfg.blockDim = dim3((unsigned)(32 * W));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclusters = 0;
  const cudaError_t oc = cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg);
  if (getenv("KZ_VERBOSE"))
    fprintf(stderr, "[kz cluster] W %d CL %d smem %zu: max active clusters %d (%s)\n", W, CL, smem, nclusters,
            cudaGetErrorString(oc));
  if (oc != cudaSuccess || nclusters < 1) {
    cudaGetLastError();
    return 0;
  }
  if (g_dry_launch) return 1;
  note_tma(ST ? 0 : a.bulk);
  if (ST) {
    const long long rows = (long long)a.P.n_systems * a.P.n_users;
    kz_hpad_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(a.P, a.NS, const_cast<float2*>(a.hpad));
  }
  if (cudaLaunchKernelEx(&cfg, kern, a) != cudaSuccess) return -1;
  if (a.mode == KZ_STOP_LOCKSTEP)
    kz_lockstep_finalize<<<(a.P.n_systems + 127) / 128, 128, 0, s>>>(a.tstop, groups, a.P.n_systems, a.O.n_outer,
                                                                     a.O.sys_converged);
  return 1;
}

// 1 launched, 0 not eligible, -1 failure
inline int cluster_try_launch(const kz_problem& P, int scheme, const kz_stop& S, const kz_rng& R, const kz_out& O,
                              int resume, char* ws, size_t ws_bytes, cudaStream_t s, int32_t* launches) {
  static const bool disabled = getenv("KZ_DISABLE_FAST") != nullptr || getenv("KZ_DISABLE_CLUSTER") != nullptr;
  if (disabled || resume || P.dtype != KZ_C64) return 0;
  if (!(scheme == KZ_GK || scheme == KZ_GRK || scheme == KZ_VR_OGRK || scheme == KZ_AHK || scheme == KZ_VR_OAHK ||
        scheme == KZ_VR_OAHK_G))
    return 0;
  const bool lockstep = S.mode == KZ_STOP_LOCKSTEP && S.epsilon == 0.0;
  const bool resid = S.mode == KZ_STOP_RESIDUAL && S.epsilon > 0.0;
  if (!(lockstep || resid) || S.max_iters < 1 || S.check_every < 1) return 0;
  // grouped vr-oahk: fixed T only (the cfg3 workload), set ids fit uint8; residual / NMSE runs take the generic kernel
  if (scheme == KZ_VR_OAHK_G && (!lockstep || P.n_users > 254 || !P.ogrp_sys || !P.ogrp_ptr)) return 0;
  if (O.nmse_trace || O.resid_trace || O.flops_trace || S.rhs_mask) return 0;
  if (!(P.flags & KZ_PROBLEM_CONTIGUOUS) || P.max_support < 1 || P.n_antennas % clu::CH != 0) return 0;
  const bool stochastic = scheme == KZ_GRK || scheme == KZ_VR_OGRK;
  if (stochastic && R.kind != KZ_RNG_PHILOX &&
      !(lockstep && R.kind == KZ_RNG_HOST_UNIFORM && R.stream_base == 0 && R.stream_len >= S.max_iters))
    return 0;
  if (ws_bytes < ls_extra_ws(P)) return 0;  // tstop only: the per-rhs state lives on chip
  int dev = 0, maxsm = 0, smsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&smsm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  // slice width: 256 antennas (8 warps, one CTA per SM) when it fits, else 128 antennas (two CTAs per SM when
  // they fit); clusters stay within 16 CTAs
  // candidates in order of preference: 32 rhs x 256-antenna CTAs, 16 rhs x 256, 16 rhs x 128 (two CTAs per
  // SM when they fit), 16 rhs x 128; clusters stay within 16 CTAs
  struct Cand { int G, W, CL, NS, pcap, rcap; size_t smem; bool two_per_sm, st; };
  // streamed (ST) candidates first when enabled: H_eff read through L1 / L2, two CTAs per SM; they need the padded
  // copy in the workspace (kz_solve_workspace_bytes_for reports it), 20-bit piece offsets and, for the aggregation
  // schemes, 16 rhs (m and y of 32 rhs do not fit the 128 registers of two CTAs per SM)
  const bool agg_scheme = scheme == KZ_AHK || scheme == KZ_VR_OAHK || scheme == KZ_VR_OAHK_G;
  Cand cands[7] = {{32, 8, 0, 0, 0, 0, 0, true, true}, {16, 8, 0, 0, 0, 0, 0, true, true},
                   {32, 8}, {16, 8}, {16, 4}, {16, 4}, {32, 4}};
  const size_t two = (size_t)(smsm / 2 - 1024);
  // KZ_CLUSTER_STREAM: 0 never, 1 (default) where it measured faster, 2 whenever eligible.  Measured same-box
  // (tools/ab_stream.sh, profiles/r02_ab_cluster_stream.log): the aggregation schemes in residual mode (cfg4
  // vr-oahk: ~2.4 iterations per rhs, so staging H_eff into shared memory was a large part of the launch) -16%;
  // cfg4 grk -1%; the fixed-T cfg3 / cfg5 aggregation runs +12..28% (H_eff re-read from L2 every iteration)
  static const int env_stream = getenv("KZ_CLUSTER_STREAM") ? atoi(getenv("KZ_CLUSTER_STREAM")) : 1;
  const bool want_stream = env_stream == 2 || (env_stream == 1 && resid && agg_scheme);
  for (int k = 0; k < 7; ++k) {
    Cand& cd = cands[k];
    cd.smem = cluster_smem_bytes(P, scheme, cd.W, cd.G, &cd.CL, &cd.NS, &cd.pcap, &cd.rcap, cd.st);
    if (k == 4) cd.two_per_sm = true;
    if (cd.st) {
      const bool ok = want_stream && !(agg_scheme && cd.G == 32) && (long long)P.n_users * cd.NS * clu::CH < (1 << 20) &&
                      ws_bytes >= cluster_hpad_offset(P) + cluster_hpad_bytes(P, cd.NS);
      if (!ok) cd.smem = ~size_t(0);
    }
  }
  static const int forced_w = getenv("KZ_CLUSTER_W") ? atoi(getenv("KZ_CLUSTER_W")) : 0;
  static const int forced_g = getenv("KZ_CLUSTER_G") ? atoi(getenv("KZ_CLUSTER_G")) : 0;
  int pick = -1;
  for (int k = 0; k < 7 && pick < 0; ++k) {
    const Cand& cd = cands[k];
    if ((forced_w && cd.W != forced_w) || (forced_g && cd.G != forced_g)) continue;
    if (cd.CL > 16 || cd.smem > (cd.two_per_sm ? two : (size_t)maxsm)) continue;
    pick = k;
  }
  static const bool verbose = getenv("KZ_VERBOSE") != nullptr;
  if (verbose)
    for (int k = 0; k < 7; ++k)
      fprintf(stderr, "[kz cluster] scheme %d K %d Nt %d: G %d W %d CL %d%s pairs %d smem %zu%s\n", scheme,
              P.n_users, P.n_antennas, cands[k].G, cands[k].W, cands[k].CL, cands[k].st ? " streamed" : "",
              cands[k].pcap, cands[k].smem == ~size_t(0) ? 0 : cands[k].smem, k == pick ? "  <- picked" : "");
  if (pick < 0) return 0;
  const int W = cands[pick].W, CL = cands[pick].CL, GG = cands[pick].G;
  const bool ST = cands[pick].st;
  const size_t smem = cands[pick].smem;
  g_cluster_dry_ws = ST ? cluster_hpad_offset(P) + cluster_hpad_bytes(P, cands[pick].NS) : ls_extra_ws(P);
  CluArgs a;
  a.P = P;
  a.bulk = bulk_staging_ok(P);
  a.R = R;
  a.O = O;
  a.mode = lockstep ? KZ_STOP_LOCKSTEP : KZ_STOP_RESIDUAL;
  a.cap = S.max_iters;
  a.every = S.check_every;
  a.eps = (float)S.epsilon;
  a.NS = cands[pick].NS;
  static const int env_nblk = getenv("KZ_CLUSTER_NBLK") ? atoi(getenv("KZ_CLUSTER_NBLK")) : 2;
  const int nb = env_nblk > 0 && W % env_nblk == 0 ? env_nblk : 2;
  a.nblk = CL > 1 ? nb : 1;  // must match the layout hint (HostBatch.slice_pairs / batch.cluster_blocks)
  a.pcap = cands[pick].pcap;
  a.rcap = cands[pick].rcap;
  a.tstop = (int32_t*)ws;
  a.hpad = ST && ws ? (const float2*)(ws + cluster_hpad_offset(P)) : nullptr;
  static const int env_order = getenv("KZ_CLUSTER_RHS_ORDER") ? atoi(getenv("KZ_CLUSTER_RHS_ORDER")) : 1;
  a.order = env_order;
  int rc = 0;
  if (ST) {
    if (GG == 32) {
      switch (scheme) {
        case KZ_GK: rc = cluster_launch<KZ_GK, 32, true>(a, W, CL, smem, s); break;
        case KZ_GRK: rc = cluster_launch<KZ_GRK, 32, true>(a, W, CL, smem, s); break;
        case KZ_VR_OGRK: rc = cluster_launch<KZ_VR_OGRK, 32, true>(a, W, CL, smem, s); break;
      }
    } else {
      switch (scheme) {
        case KZ_GK: rc = cluster_launch<KZ_GK, 16, true>(a, W, CL, smem, s); break;
        case KZ_GRK: rc = cluster_launch<KZ_GRK, 16, true>(a, W, CL, smem, s); break;
        case KZ_VR_OGRK: rc = cluster_launch<KZ_VR_OGRK, 16, true>(a, W, CL, smem, s); break;
        case KZ_AHK: rc = cluster_launch<KZ_AHK, 16, true>(a, W, CL, smem, s); break;
        case KZ_VR_OAHK: rc = cluster_launch<KZ_VR_OAHK, 16, true>(a, W, CL, smem, s); break;
      }
    }
  } else if (GG == 32) {
    switch (scheme) {
      case KZ_GK: rc = cluster_launch<KZ_GK, 32, false>(a, W, CL, smem, s); break;
      case KZ_GRK: rc = cluster_launch<KZ_GRK, 32, false>(a, W, CL, smem, s); break;
      case KZ_VR_OGRK: rc = cluster_launch<KZ_VR_OGRK, 32, false>(a, W, CL, smem, s); break;
      case KZ_AHK: rc = cluster_launch<KZ_AHK, 32, false>(a, W, CL, smem, s); break;
      case KZ_VR_OAHK: rc = cluster_launch<KZ_VR_OAHK, 32, false>(a, W, CL, smem, s); break;
      case KZ_VR_OAHK_G: rc = cluster_launch<KZ_VR_OAHK_G, 32, false>(a, W, CL, smem, s); break;
    }
  } else {
    switch (scheme) {
      case KZ_GK: rc = cluster_launch<KZ_GK, 16, false>(a, W, CL, smem, s); break;
      case KZ_GRK: rc = cluster_launch<KZ_GRK, 16, false>(a, W, CL, smem, s); break;
      case KZ_VR_OGRK: rc = cluster_launch<KZ_VR_OGRK, 16, false>(a, W, CL, smem, s); break;
      case KZ_AHK: rc = cluster_launch<KZ_AHK, 16, false>(a, W, CL, smem, s); break;
      case KZ_VR_OAHK: rc = cluster_launch<KZ_VR_OAHK, 16, false>(a, W, CL, smem, s); break;
      case KZ_VR_OAHK_G: rc = cluster_launch<KZ_VR_OAHK_G, 16, false>(a, W, CL, smem, s); break;
    }
  }
  if (rc == 1) *launches = (lockstep ? 2 : 1) + (ST ? 1 : 0);
  return rc;
}

}  // namespace kz
