// On-device input preparation for the BASELINE channel model: the packed VR rows of
// every system from its user drop, and the VR partition, so cfg4/cfg5-sized batches are not limited by
// host-side numpy generation and the 16 GiB PCIe copy of H_eff.
//
//   kz_channel_synth  <- channel.generate / _entries (paper_2501_10689_b200/channel.py): near-field LoS entry
//                        lambda/(4 pi r_n) exp(-j 2 pi r_n / lambda) on a contiguous VR, unit-norm column,
//                        e_i = ||h_i||^2 + xi (solvers.py:90)
//   kz_partition_*    <- build_partition (pkg/src/kaczprec/vrgraph.py:31-114): interval-overlap graph,
//                        minimum-residual-degree greedy MIS with lowest-index tie-break (vrgraph.py:43-56),
//                        coupled sets X_k = N(k) + {k}, N ascending, |union of N supports|
#pragma once

#include "kz_common.cuh"

namespace kz {

// one warp per row (b, i): fp64 entries, warp-reduced norm, normalised values in the output dtype
template <class T>
__global__ void kz_channel_synth_kernel(kz_drop D, const int64_t* row_val_ptr, T* heff, double* row_energy) {
  const int lane = threadIdx.x & 31;
  const size_t row = (size_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const size_t rows = (size_t)D.n_systems * D.n_users;
  if (row >= rows) return;
  const int b = (int)(row / D.n_users);
  const double lam = D.wavelength[b];
  const double r0 = D.r0[row], th = D.theta[row];
  const int s = D.vr_start[row], L = D.vr_len[row];
  const double half = (D.n_antennas - 1) / 2.0;
  const double ca = cos(M_PI / 2.0 - th);  // cos of the angle to the array axis
  const double amp0 = 4.0 * M_PI;
  T* out = heff + row_val_ptr[row];
  double ss = 0.0;
  for (int e = lane; e < L; e += 32) {
    const double x = ((double)(s + e) - half) * D.element_spacing;
    const double r = sqrt(r0 * r0 + x * x - 2.0 * x * r0 * ca);
    const double amp = lam / (amp0 * r);
    const double ph = (2.0 * M_PI * r) / lam;
    double sn, cs;
    sincos(ph, &sn, &cs);
    const double hx = amp * cs, hy = -amp * sn;
    ss = fma(hx, hx, fma(hy, hy, ss));
  }
  ss = warp_sum(ss);
  const double nrm = sqrt(ss);
  double e2 = 0.0;
  for (int e = lane; e < L; e += 32) {  // recompute instead of staging: rows are up to Nt long
    const double x = ((double)(s + e) - half) * D.element_spacing;
    const double r = sqrt(r0 * r0 + x * x - 2.0 * x * r0 * ca);
    const double amp = lam / (amp0 * r);
    const double ph = (2.0 * M_PI * r) / lam;
    double sn, cs;
    sincos(ph, &sn, &cs);
    const double hx = (amp * cs) / nrm, hy = (-(amp * sn)) / nrm;
    out[e] = from_d2<T>(make_double2(hx, hy));
    e2 = fma(hx, hx, fma(hy, hy, e2));  // energy of the fp64 row (as the host packer computes it)
  }
  e2 = warp_sum(e2);
  if (lane == 0) row_energy[row] = e2 + D.reg[b];
}

// one CTA (warp 0 runs the greedy loop) per system; adjacency as bitsets in shared memory
// mode 0: counts (coupled_cnt, orth_cnt, non_union_size, inset); mode 1: fill the index lists
__global__ void kz_partition_kernel(kz_drop D, int mode, int32_t* coupled_cnt, int32_t* orth_cnt,
                                    int32_t* non_union_size, uint8_t* inset, const int32_t* coupled_ptr,
                                    const int32_t* orth_ptr, const int32_t* non_ptr, int32_t* coupled_idx,
                                    int32_t* orth_idx, int32_t* non_idx) {
  extern __shared__ __align__(16) unsigned char psm[];
  const int b = blockIdx.x, K = D.n_users, KW = (K + 31) / 32;
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31;
  uint32_t* adj = (uint32_t*)psm;                 // [K][KW]
  uint32_t* alive = adj + (size_t)K * KW;         // [KW]
  int* deg = (int*)(alive + KW);                  // [K]
  int* st = deg + K;                              // [K]
  int* en = st + K;                               // [K] exclusive end
  uint32_t* cover = (uint32_t*)(en + K);          // [Nt / 32 + 1] antennas covered by N
  uint8_t* ins = (uint8_t*)(cover + D.n_antennas / 32 + 1);  // [K]
  const size_t r0 = (size_t)b * K;
  for (int i = tid; i < K; i += nthr) {
    st[i] = D.vr_start[r0 + i];
    en[i] = st[i] + D.vr_len[r0 + i];
  }
  __syncthreads();
  for (int e = tid; e < K * KW; e += nthr) {  // overlap graph, no self loops
    const int i = e / KW, q = e % KW;
    uint32_t wd = 0;
    for (int t = 0; t < 32; ++t) {
      const int j = 32 * q + t;
      if (j < K && j != i && st[i] < en[j] && st[j] < en[i]) wd |= 1u << t;
    }
    adj[e] = wd;
  }
  __syncthreads();
  if (tid < 32) {
    for (int q = lane; q < KW; q += 32) alive[q] = (q == KW - 1 && (K & 31)) ? (1u << (K & 31)) - 1 : 0xFFFFFFFFu;
    for (int i = lane; i < K; i += 32) {
      int d = 0;
      for (int q = 0; q < KW; ++q) d += __popc(adj[i * KW + q]);
      deg[i] = d;
      ins[i] = 2;
    }
    __syncwarp();
    // greedy MIS: smallest residual degree, ties by lowest index (vrgraph.py:52-55)
    while (true) {
      long long best = 0x7fffffffffffffffLL;
      for (int i = lane; i < K; i += 32)
        if ((alive[i >> 5] >> (i & 31)) & 1u) {
          const long long key = (long long)deg[i] * (K + 1) + i;
          best = key < best ? key : best;
        }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const long long ob = __shfl_xor_sync(FULL, best, o);
        best = ob < best ? ob : best;
      }
      if (best == 0x7fffffffffffffffLL) break;
      const int v = (int)(best % (K + 1));
      // remove v and its alive neighbours; every removed vertex decrements its alive neighbours' degrees
      __syncwarp();
      if (lane == 0) ins[v] = 1;
      for (int q = 0; q < KW; ++q) {
        uint32_t rm = (adj[v * KW + q] & alive[q]) | (q == (v >> 5) ? (1u << (v & 31)) : 0u);
        __syncwarp();
        if (lane == 0) alive[q] &= ~rm;
        __syncwarp();
        while (rm) {
          const int u = 32 * q + __ffs(rm) - 1;
          rm &= rm - 1;
          for (int i = lane; i < K; i += 32)
            if (((alive[i >> 5] >> (i & 31)) & 1u) && ((adj[u * KW + (i >> 5)] >> (i & 31)) & 1u)) deg[i] -= 1;
          __syncwarp();
        }
      }
    }
  }
  __syncthreads();
  if (mode == 0) {
    const int nw = D.n_antennas / 32 + 1;
    for (int q = tid; q < nw; q += nthr) cover[q] = 0;
    __syncthreads();
    for (int i = tid; i < K; i += nthr) {
      int c = 1;
      for (int q = 0; q < KW; ++q) c += __popc(adj[i * KW + q]);
      coupled_cnt[r0 + i] = c;
      inset[r0 + i] = ins[i];
      if (ins[i] == 2)
        for (int n = st[i]; n < en[i]; ++n) atomicOr(&cover[n >> 5], 1u << (n & 31));
    }
    __syncthreads();
    if (tid < 32) {
      int o = 0, u = 0;
      for (int i = lane; i < K; i += 32) o += ins[i] == 1;
      for (int q = lane; q < nw; q += 32) u += __popc(cover[q]);
      o = warp_sum(o);
      u = warp_sum(u);
      if (lane == 0) {
        orth_cnt[b] = o;
        non_union_size[b] = u;
      }
    }
    return;
  }
  // mode 1: index lists, ascending
  for (int i = tid; i < K; i += nthr) {
    int p = coupled_ptr[r0 + i];
    for (int j = 0; j < K; ++j)
      if (j == i || ((adj[i * KW + (j >> 5)] >> (j & 31)) & 1u)) coupled_idx[p++] = j;
  }
  if (tid == 0) {
    int po = orth_ptr[b], pn = non_ptr[b];
    for (int i = 0; i < K; ++i) {
      if (ins[i] == 1) orth_idx[po++] = i;
      else non_idx[pn++] = i;
    }
  }
}

inline size_t partition_smem(int K, int Nt) {
  const int KW = (K + 31) / 32;
  return (size_t)K * KW * 4 + KW * 4 + 3 * (size_t)K * 4 + ((size_t)Nt / 32 + 1) * 4 + K + 16;
}

}  // namespace kz
