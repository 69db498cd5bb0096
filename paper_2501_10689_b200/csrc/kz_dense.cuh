// Direct RZF solve (K2) and precoder epilogue (K3), one CTA per system.
//
//   kz_rzf_kernel      <- rzf.py:38-83  (Gram, Cholesky, V = Gram^{-1}, F = beta H V)
//   kz_epilogue_kernel <- assembly.py:51-92 + metrics.py:44-78
//
// H is never formed densely: the Gram is accumulated over pairwise support
// intersections and F = H V over the rows covering each antenna (the
// VR-blocked product of assemble_vr with one-antenna blocks).  The epilogue
// never materialises F unless asked: the NMSE against F_ref = beta_ref H V_ref
// is ||H (beta_ref V_ref - beta V)||_F / ||beta_ref H V_ref||_F and the rate
// cross terms are H^H F = beta (H^H H) V.
#pragma once

#include "kz_common.cuh"

namespace kz {

constexpr int DENSE_THREADS = 256;

struct RowView {
  const int32_t* seg_ptr;
  const int32_t* seg_start;
  const int32_t* seg_len;
  const int64_t* val_ptr;
};

// heff index of antenna n in row r's packed values, or -1
__device__ __forceinline__ int64_t row_pos(const RowView& R, size_t r, int n) {
  int s0 = R.seg_ptr[r], s1 = R.seg_ptr[r + 1];
  int64_t v = R.val_ptr[r];
  for (int s = s0; s < s1; ++s) {
    int st = R.seg_start[s], ln = R.seg_len[s];
    if (n < st) return -1;
    if (n < st + ln) return v + (n - st);
    v += ln;
  }
  return -1;
}

template <class T> __device__ __forceinline__ double2 ld_d2(const void* base, int64_t i) {
  return to_d2(((const T*)base)[i]);
}

// (H^H H)_{ij} over the intersection of two segment lists, accumulated in double
template <class T>
__device__ double2 gram_entry(const RowView& R, const void* heff, size_t ri, size_t rj) {
  int a = R.seg_ptr[ri], a1 = R.seg_ptr[ri + 1];
  int b = R.seg_ptr[rj], b1 = R.seg_ptr[rj + 1];
  int64_t va = R.val_ptr[ri], vb = R.val_ptr[rj];
  double re = 0.0, im = 0.0;
  while (a < a1 && b < b1) {
    int sa = R.seg_start[a], la = R.seg_len[a];
    int sb = R.seg_start[b], lb = R.seg_len[b];
    int lo = max(sa, sb), hi = min(sa + la, sb + lb);
    for (int n = lo; n < hi; ++n) {
      double2 x = ld_d2<T>(heff, va + (n - sa)), y = ld_d2<T>(heff, vb + (n - sb));
      re = fma(x.x, y.x, re);
      re = fma(x.y, y.y, re);
      im = fma(x.x, y.y, im);
      im = fma(-x.y, y.x, im);
    }
    if (sa + la <= sb + lb) { va += la; ++a; } else { vb += lb; ++b; }
  }
  return make_double2(re, im);
}

__device__ inline double block_reduce_sum(double v, double* red) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < nw; ++i) t += red[i];
  __syncthreads();
  return t;
}

// Per-antenna assembly.  For every antenna n and column c computes
//   a = sum_{i covers n} h_i[n] (sa * Va[i][c] - sb * Vb[i][c])      (Vb optional)
// optionally stores a (as TF) into f[n][c], and returns block-reduced ||a||^2
// and, if Vb given, ||sb * H Vb||^2 in *ref_sq.
template <class TH, class TV, class TF>
__device__ double assemble(const kz_problem& P, int b, const TV* Va, double sa, const double2* Vb, double sb, TF* f,
                           double* ref_sq, double* red) {
  const int K = P.n_users, Nt = P.n_antennas;
  RowView R{P.row_seg_ptr, P.seg_start, P.seg_len, P.row_val_ptr};
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double ss = 0.0, rs = 0.0;
  for (int n = warp; n < Nt; n += nw) {
    for (int c0 = 0; c0 < K; c0 += 32) {
      int c = c0 + lane;
      double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
      for (int i = 0; i < K; ++i) {  // ascending users covering antenna n
        int64_t pos = row_pos(R, (size_t)b * K + i, n);
        if (pos < 0 || c >= K) continue;
        double2 h = ld_d2<TH>(P.heff, pos);
        double2 x = to_d2(Va[(size_t)i * K + c]);
        x.x *= sa;
        x.y *= sa;
        if (Vb) {
          double2 y = Vb[(size_t)i * K + c];
          y.x *= sb;
          y.y *= sb;
          br = fma(h.x, y.x, br);
          br = fma(-h.y, y.y, br);
          bi = fma(h.x, y.y, bi);
          bi = fma(h.y, y.x, bi);
          x.x -= y.x;
          x.y -= y.y;
        }
        ar = fma(h.x, x.x, ar);
        ar = fma(-h.y, x.y, ar);
        ai = fma(h.x, x.y, ai);
        ai = fma(h.y, x.x, ai);
      }
      if (c < K) {
        if (f) f[(size_t)n * K + c] = from_d2<TF>(make_double2(ar, ai));
        ss += ar * ar + ai * ai;
        rs += br * br + bi * bi;
      }
    }
  }
  ss = block_reduce_sum(ss, red);
  if (Vb) *ref_sq = block_reduce_sum(rs, red);
  return ss;
}

// ---------------------------------------------------------------- K2: RZF
template <class TH>
__global__ void __launch_bounds__(DENSE_THREADS) kz_rzf_kernel(kz_problem P, double* v_out, double* f_out,
                                                               double* beta_out, uint8_t* pd_ok, double2* ws) {
  const int b = blockIdx.x;
  const int K = P.n_users, Nt = P.n_antennas;
  RowView R{P.row_seg_ptr, P.seg_start, P.seg_len, P.row_val_ptr};
  double2* G = ws + (size_t)b * 2 * K * K;  // Gram -> L (lower)
  double2* Z = G + (size_t)K * K;           // L^{-1}
  __shared__ double red[32];
  __shared__ int s_bad;
  __shared__ double s_d;
  const double reg = P.reg[b];

  // Gram, lower triangle (rzf.py:38-40)
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
    int i = e / K, j = e % K;
    if (j > i) continue;
    double2 g = gram_entry<TH>(R, P.heff, (size_t)b * K + i, (size_t)b * K + j);
    if (i == j) { g.x += reg; g.y = 0.0; }
    G[(size_t)i * K + j] = g;
  }
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  // right-looking Cholesky, lower (scipy cho_factor(lower=True) -> LAPACK potrf)
  for (int k = 0; k < K; ++k) {
    if (threadIdx.x == 0) {
      double d = G[(size_t)k * K + k].x;
      if (!(d > 0.0)) { s_bad = 1; d = 1.0; }
      s_d = sqrt(d);
      G[(size_t)k * K + k] = make_double2(s_d, 0.0);
    }
    __syncthreads();
    double d = s_d;
    for (int i = k + 1 + threadIdx.x; i < K; i += blockDim.x) {
      double2 x = G[(size_t)i * K + k];
      G[(size_t)i * K + k] = make_double2(x.x / d, x.y / d);
    }
    __syncthreads();
    int m = K - k - 1;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      int i = k + 1 + e / m, j = k + 1 + e % m;
      if (j > i) continue;
      double2 li = G[(size_t)i * K + k], lj = G[(size_t)j * K + k];
      double2 g = G[(size_t)i * K + j];
      g.x -= li.x * lj.x + li.y * lj.y;  // g -= li * conj(lj)
      g.y -= li.y * lj.x - li.x * lj.y;
      G[(size_t)i * K + j] = g;
    }
    __syncthreads();
  }
  if (pd_ok && threadIdx.x == 0) pd_ok[b] = s_bad ? 0 : 1;
  // Z = L^{-1}, one thread per column (forward substitution)
  for (int c = threadIdx.x; c < K; c += blockDim.x) {
    for (int i = 0; i < c; ++i) Z[(size_t)i * K + c] = make_double2(0.0, 0.0);
    for (int i = c; i < K; ++i) {
      double re = i == c ? 1.0 : 0.0, im = 0.0;
      for (int k = c; k < i; ++k) {
        double2 l = G[(size_t)i * K + k], z = Z[(size_t)k * K + c];
        re -= l.x * z.x - l.y * z.y;
        im -= l.x * z.y + l.y * z.x;
      }
      double lii = G[(size_t)i * K + i].x;
      Z[(size_t)i * K + c] = make_double2(re / lii, im / lii);
    }
  }
  __syncthreads();
  // V = Z^H Z = (L L^H)^{-1}  (cho_solve(., I), rzf.py:60-66)
  double2* V = (double2*)v_out + (size_t)b * K * K;
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
    int i = e / K, j = e % K;
    double re = 0.0, im = 0.0;
    for (int k = max(i, j); k < K; ++k) {
      double2 a = Z[(size_t)k * K + i], c = Z[(size_t)k * K + j];
      re = fma(a.x, c.x, re);
      re = fma(a.y, c.y, re);
      im = fma(a.x, c.y, im);
      im = fma(-a.y, c.x, im);
    }
    V[e] = make_double2(re, im);
  }
  __syncthreads();
  // beta = 1/||H V||_F, F = beta H V (rzf.py:77-83)
  double2* F = f_out ? (double2*)f_out + (size_t)b * Nt * K : nullptr;
  double ss = assemble<TH, double2, double2>(P, b, V, 1.0, nullptr, 0.0, F, nullptr, red);
  double beta = 1.0 / sqrt(ss);
  if (F)
    for (size_t e = threadIdx.x; e < (size_t)Nt * K; e += blockDim.x) {
      double2 x = F[e];
      F[e] = make_double2(x.x * beta, x.y * beta);
    }
  if (beta_out && threadIdx.x == 0) beta_out[b] = beta;
}

// ---------------------------------------------------------------- K3: epilogue
template <class T>
__global__ void __launch_bounds__(DENSE_THREADS) kz_epilogue_kernel(kz_problem P, const T* v, T* f_out, const double* v_ref,
                                                                    const double* beta_ref, const double* snr_linear,
                                                                    double* beta_out, double* nmse_out, double* rates_out,
                                                                    double* sum_rate_out, double2* ws) {
  const int b = blockIdx.x;
  const int K = P.n_users, Nt = P.n_antennas;
  RowView R{P.row_seg_ptr, P.seg_start, P.seg_len, P.row_val_ptr};
  __shared__ double red[32];
  const T* Vb = v + (size_t)b * K * K;
  // pass 1: ||H V||_F -> beta (assembly.py:51-56)
  double ss = assemble<T, T, T>(P, b, Vb, 1.0, nullptr, 0.0, nullptr, nullptr, red);
  const double beta = 1.0 / sqrt(ss);
  if (beta_out && threadIdx.x == 0) beta_out[b] = beta;
  // pass 2: F = beta H V (stored on request) and NMSE vs beta_ref H V_ref
  T* F = f_out ? f_out + (size_t)b * Nt * K : nullptr;
  if (F) assemble<T, T, T>(P, b, Vb, beta, nullptr, 0.0, F, nullptr, red);
  if (v_ref && nmse_out) {
    double ref_sq = 0.0;
    const double2* Vr = (const double2*)v_ref + (size_t)b * K * K;
    double d2 = assemble<T, T, T>(P, b, Vb, beta, Vr, beta_ref[b], (T*)nullptr, &ref_sq, red);
    if (threadIdx.x == 0) nmse_out[b] = sqrt(d2) / sqrt(ref_sq);
  }
  if (!snr_linear) return;
  // rates (metrics.py:54-78): cross = H^H F = beta Gram0 V
  double2* G = ws + (size_t)b * K * K;
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
    int i = e / K, j = e % K;
    G[e] = gram_entry<T>(R, P.heff, (size_t)b * K + i, (size_t)b * K + j);
  }
  __syncthreads();
  const double noise = 1.0 / snr_linear[b];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double rsum = 0.0;
  for (int k = warp; k < K; k += nw) {
    double sig = 0.0, tot = 0.0;
    for (int c0 = 0; c0 < K; c0 += 32) {
      int c = c0 + lane;
      double re = 0.0, im = 0.0;
      if (c < K)
        for (int j = 0; j < K; ++j) {
          double2 g = G[(size_t)k * K + j];
          double2 x = to_d2(Vb[(size_t)j * K + c]);
          re = fma(g.x, x.x, re);
          re = fma(-g.y, x.y, re);
          im = fma(g.x, x.y, im);
          im = fma(g.y, x.x, im);
        }
      double p = c < K ? np_abs2(re * beta, im * beta) : 0.0;
      if (c == k) sig = p;
      tot += p;
    }
    tot = warp_sum(tot);
    sig = warp_sum(sig);
    if (lane == 0) {
      double rate = log2(1.0 + sig / ((tot - sig) + noise));
      if (rates_out) rates_out[(size_t)b * K + k] = rate;
      rsum += rate;
    }
  }
  rsum = block_reduce_sum(rsum, red);
  if (sum_rate_out && threadIdx.x == 0) sum_rate_out[b] = rsum;
}

}  // namespace kz

namespace kz {

// ---------------------------------------------------------------- K3 fast path (contiguous VRs)
// One CTA per system.  Rows are ranked by VR start so the rows covering antenna n
// form a short window found by two binary searches; F = H V is assembled per
// antenna with lanes over the K columns.  Pass 1 gives beta = 1/||HV||_F, pass 2
// stores F = beta H V and accumulates ||beta_ref H V_ref - beta H V||^2 directly
// (no cancellation), pass 3 forms H^H F over each user's VR for the Eq. (7) rates.
template <class T>
__global__ void __launch_bounds__(DENSE_THREADS) kz_epilogue_contig_kernel(
    kz_problem P, const T* v, T* f_out, const double* v_ref, const double* beta_ref, const double* snr_linear,
    double* beta_out, double* nmse_out, double* rates_out, double* sum_rate_out, T* fws) {
  using R = typename Cx<T>::real;
  extern __shared__ __align__(16) unsigned char sm[];
  const int b = blockIdx.x, K = P.n_users, Nt = P.n_antennas;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int* st = (int*)sm;            // starts, original order
  int* ln = st + K;              // lengths
  int* ord = ln + K;             // rows ranked by start
  int* ss = ord + K;             // sorted starts
  long long* off = (long long*)(ss + K + (K & 1));
  __shared__ double red[32];
  __shared__ int s_lmax;
  for (int i = threadIdx.x; i < K; i += blockDim.x) {
    size_t r = (size_t)b * K + i;
    int sg = P.row_seg_ptr[r];
    st[i] = P.seg_start[sg];
    ln[i] = P.seg_len[sg];
    off[i] = P.row_val_ptr[r];
  }
  if (threadIdx.x == 0) s_lmax = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < K; i += blockDim.x) {
    int rk = 0;
    for (int j = 0; j < K; ++j) rk += (st[j] < st[i]) || (st[j] == st[i] && j < i);
    ord[rk] = i;
    ss[rk] = st[i];
    atomicMax(&s_lmax, ln[i]);
  }
  __syncthreads();
  const int lmax = s_lmax;
  const T* H = (const T*)P.heff;
  const T* V = v + (size_t)b * K * K;
  const double2* Vr = v_ref ? (const double2*)v_ref + (size_t)b * K * K : nullptr;
  auto window = [&](int n, int& lo, int& hi) {  // sorted positions with n - lmax < start <= n
    int a0 = 0, a1 = K;
    while (a0 < a1) { int m = (a0 + a1) >> 1; if (ss[m] <= n) a0 = m + 1; else a1 = m; }
    hi = a0;
    a0 = 0; a1 = hi;
    while (a0 < a1) { int m = (a0 + a1) >> 1; if (ss[m] <= n - lmax) a0 = m + 1; else a1 = m; }
    lo = a0;
  };
  // pass 1: ||H V||_F^2
  double s1 = 0.0;
  for (int n = warp; n < Nt; n += nw) {
    int lo, hi;
    window(n, lo, hi);
    for (int c0 = 0; c0 < K; c0 += 32) {
      const int c = c0 + lane;
      R fr = 0, fi = 0;
      for (int j = lo; j < hi; ++j) {
        const int i = ord[j];
        if (n >= st[i] + ln[i]) continue;
        const T h = H[off[i] + (n - st[i])];
        if (c < K) {
          const T x = V[(size_t)i * K + c];
          fr = fma(h.x, x.x, fr); fr = fma(-h.y, x.y, fr);
          fi = fma(h.x, x.y, fi); fi = fma(h.y, x.x, fi);
        }
      }
      s1 += (double)fr * fr + (double)fi * fi;
    }
  }
  s1 = block_reduce_sum(s1, red);
  const double beta = 1.0 / sqrt(s1);
  if (beta_out && threadIdx.x == 0) beta_out[b] = beta;
  // pass 2: F = beta H V (stored), NMSE against beta_ref H V_ref
  T* F = f_out ? f_out + (size_t)b * Nt * K : fws + (size_t)b * Nt * K;
  const double br = Vr ? beta_ref[b] : 0.0;
  double e2 = 0.0, r2 = 0.0;
  for (int n = warp; n < Nt; n += nw) {
    int lo, hi;
    window(n, lo, hi);
    for (int c0 = 0; c0 < K; c0 += 32) {
      const int c = c0 + lane;
      R fr = 0, fi = 0;
      double gr = 0.0, gi = 0.0;
      for (int j = lo; j < hi; ++j) {
        const int i = ord[j];
        if (n >= st[i] + ln[i]) continue;
        const T h = H[off[i] + (n - st[i])];
        if (c < K) {
          const T x = V[(size_t)i * K + c];
          fr = fma(h.x, x.x, fr); fr = fma(-h.y, x.y, fr);
          fi = fma(h.x, x.y, fi); fi = fma(h.y, x.x, fi);
          if (Vr) {
            const double2 y = Vr[(size_t)i * K + c];
            const double hx = h.x, hy = h.y;
            gr = fma(hx, y.x, gr); gr = fma(-hy, y.y, gr);
            gi = fma(hx, y.y, gi); gi = fma(hy, y.x, gi);
          }
        }
      }
      if (c < K) {
        const double ox = beta * fr, oy = beta * fi;
        F[(size_t)n * K + c] = from_d2<T>(make_double2(ox, oy));
        if (Vr) {
          const double dx = br * gr - ox, dy = br * gi - oy;
          e2 += dx * dx + dy * dy;
          r2 += br * br * (gr * gr + gi * gi);
        }
      }
    }
  }
  if (Vr) {
    e2 = block_reduce_sum(e2, red);
    r2 = block_reduce_sum(r2, red);
    if (nmse_out && threadIdx.x == 0) nmse_out[b] = sqrt(e2) / sqrt(r2);
  }
  if (!snr_linear) return;
  __syncthreads();  // F visible to the block
  // pass 3: Eq. (7) rates from cross = H^H F over each user's VR (metrics.py:74-77)
  const double noise = 1.0 / snr_linear[b];
  double rsum = 0.0;
  for (int k = warp; k < K; k += nw) {
    double sig = 0.0, tot = 0.0;
    for (int c0 = 0; c0 < K; c0 += 32) {
      const int c = c0 + lane;
      double re = 0.0, im = 0.0;
      if (c < K)
        for (int j = 0; j < ln[k]; ++j) {
          const double2 h = to_d2(H[off[k] + j]);
          const double2 x = to_d2(F[(size_t)(st[k] + j) * K + c]);
          re = fma(h.x, x.x, re); re = fma(h.y, x.y, re);
          im = fma(h.x, x.y, im); im = fma(-h.y, x.x, im);
        }
      const double pw = c < K ? np_abs2(re, im) : 0.0;
      if (c == k) sig = pw;
      tot += pw;
    }
    tot = warp_sum(tot);
    sig = warp_sum(sig);
    if (lane == 0) {
      const double rate = log2(1.0 + sig / ((tot - sig) + noise));
      if (rates_out) rates_out[(size_t)b * K + k] = rate;
      rsum += rate;
    }
  }
  rsum = block_reduce_sum(rsum, red);
  if (sum_rate_out && threadIdx.x == 0) sum_rate_out[b] = rsum;
}

inline size_t epilogue_contig_smem(int K) { return (size_t)4 * K * 4 + 8 + (size_t)8 * K + 64; }

}  // namespace kz
