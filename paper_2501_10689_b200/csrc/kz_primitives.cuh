// Single-system step primitives (the reference's per-call API, solvers.py:143-332) on one right-hand side
// whose state (col, coef, resid) lives in device memory.  They are the per-step building blocks the
// reference composes in InstanceRun.step; the throughput path fuses them inside the kz_solve kernels, these
// serve callers that drive a scheme one primitive at a time.  One CTA per call; the complex arithmetic
// follows numpy where it fixes the result bitwise (scalar x array products as
// re = fma(ar, br, -(ai bi)), im = fma(ar, bi, ai br); the aggregation vector accumulated per antenna over
// the rows in the caller's (ascending) order, §10.5); dot products are fixed-order tree sums.
#pragma once

#include "kz_common.cuh"

namespace kz {

constexpr int PRIM_THREADS = 256;

// numpy scalar * array element: a scalar, b array element
template <class T> __device__ __forceinline__ T np_smul(T a, T b) {
  return Cx<T>::make(fma(a.x, b.x, -(a.y * b.y)), fma(a.x, b.y, a.y * b.x));
}

struct PrimRow {  // row r = b*K + i of the packed problem
  int seg0, seg1;
  long long val0;
};

__device__ __forceinline__ PrimRow prim_row(const kz_problem& P, int b, int i) {
  const size_t r = (size_t)b * P.n_users + i;
  return {P.row_seg_ptr[r], P.row_seg_ptr[r + 1], (long long)P.row_val_ptr[r]};
}

// r_i = s_i - h_i^H col - reg coef_i for i in rows (solvers.py:143-170); warp per row.
// dense = 1: the h_adj @ col form (-dot - reg coef, then +1 on the rhs row, :149-153).
template <class T>
__global__ void __launch_bounds__(PRIM_THREADS) kz_prim_refresh(kz_problem P, int b, int rhs, const T* col,
                                                                const T* coef, T* resid, const int32_t* rows,
                                                                int n_rows, int dense) {
  using R = typename Cx<T>::real;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const T* heff = (const T*)P.heff;
  const R reg = (R)P.reg[b];
  for (int q = w; q < n_rows; q += nw) {
    const int i = rows ? rows[q] : q;
    const PrimRow pr = prim_row(P, b, i);
    R dx = 0, dy = 0;
    long long off = pr.val0;
    for (int sg = pr.seg0; sg < pr.seg1; ++sg) {
      const int s = P.seg_start[sg], L = P.seg_len[sg];
      for (int e = lane; e < L; e += 32) {
        const T h = heff[off + e], m = col[s + e];
        dx = fma(h.x, m.x, dx);
        dx = fma(h.y, m.y, dx);
        dy = fma(h.x, m.y, dy);
        dy = fma(-h.y, m.x, dy);
      }
      off += L;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      dx += __shfl_xor_sync(FULL, dx, o);
      dy += __shfl_xor_sync(FULL, dy, o);
    }
    if (lane == 0) {
      const T c = coef[i];
      T r;
      if (dense) {
        r = Cx<T>::make(-dx - reg * c.x, -dy - reg * c.y);
        if (i == rhs) r.x += (R)1;
      } else {
        const R t = i == rhs ? (R)1 : (R)0;
        r = Cx<T>::make((t - dx) - reg * c.x, ((R)0 - dy) - reg * c.y);
      }
      resid[i] = r;
    }
  }
}

// Projections onto rows in order (solvers.py:173-188 for one row, :312-332 for an orthogonal block):
// gamma = resid_i / e_i; col[Gamma_i] += gamma h_i; coef_i += gamma; resid_i = 0.  Rows are applied one
// after another (a barrier between rows), so the result is the reference's even if supports overlap.
template <class T>
__global__ void __launch_bounds__(PRIM_THREADS) kz_prim_project(kz_problem P, int b, T* col, T* coef, T* resid,
                                                                const int32_t* rows, int n_rows) {
  using R = typename Cx<T>::real;
  const T* heff = (const T*)P.heff;
  __shared__ T gam;
  for (int q = 0; q < n_rows; ++q) {
    const int i = rows[q];
    if (threadIdx.x == 0) {
      const R e = (R)P.row_energy[(size_t)b * P.n_users + i];
      const T r = resid[i];
      gam = Cx<T>::make(r.x / e, r.y / e);
    }
    __syncthreads();
    const T g = gam;
    const PrimRow pr = prim_row(P, b, i);
    long long off = pr.val0;
    for (int sg = pr.seg0; sg < pr.seg1; ++sg) {
      const int s = P.seg_start[sg], L = P.seg_len[sg];
      for (int e = threadIdx.x; e < L; e += blockDim.x) col[s + e] = cadd(col[s + e], np_smul(g, heff[off + e]));
      off += L;
    }
    if (threadIdx.x == 0) {
      coef[i] = cadd(coef[i], g);
      resid[i] = Cx<T>::make(0, 0);
    }
    __syncthreads();
  }
}

// Aggregated projection (solvers.py:257-309): num = phi_rows^H resid_rows; y = sum_i phi_i h_i accumulated per
// antenna over the rows in order; den = ||y||^2 + reg ||phi_rows||^2; den == 0 -> no step (stepped = 0);
// else gamma = num / den, col[span] += gamma y[span] (span = the union list, or every antenna when
// span == NULL), coef[rows] += gamma phi_rows.  y lives in dynamic shared memory (Nt complex).
template <class T>
__global__ void __launch_bounds__(PRIM_THREADS) kz_prim_ahk(kz_problem P, int b, T* col, T* coef, const T* resid,
                                                            const T* phi, const int32_t* rows, int n_rows,
                                                            const int32_t* span, int n_span, int32_t* stepped) {
  using R = typename Cx<T>::real;
  extern __shared__ __align__(16) unsigned char sm[];
  T* y = (T*)sm;
  __shared__ R red[3][PRIM_THREADS / 32];
  __shared__ T gam;
  __shared__ int go;
  const int Nt = P.n_antennas, tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
  const T* heff = (const T*)P.heff;
  for (int n = tid; n < Nt; n += blockDim.x) y[n] = Cx<T>::make(0, 0);
  __syncthreads();
  for (int q = 0; q < n_rows; ++q) {  // ascending rows: the reference's scatter order (bitwise, §10.5)
    const int i = rows[q];
    const T f = phi[i];
    const PrimRow pr = prim_row(P, b, i);
    long long off = pr.val0;
    for (int sg = pr.seg0; sg < pr.seg1; ++sg) {
      const int s = P.seg_start[sg], L = P.seg_len[sg];
      for (int e = tid; e < L; e += blockDim.x) y[s + e] = cadd(y[s + e], np_smul(f, heff[off + e]));
      off += L;
    }
    __syncthreads();
  }
  R yy = 0, pp = 0, nx = 0, ny = 0;
  for (int n = tid; n < Nt; n += blockDim.x) yy += y[n].x * y[n].x + y[n].y * y[n].y;
  for (int q = tid; q < n_rows; q += blockDim.x) {
    const int i = rows[q];
    const T f = phi[i], r = resid[i];
    pp += f.x * f.x + f.y * f.y;
    nx = fma(f.x, r.x, fma(f.y, r.y, nx));  // vdot: conj(phi) r
    ny = fma(f.x, r.y, fma(-f.y, r.x, ny));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    yy += __shfl_xor_sync(FULL, yy, o);
    pp += __shfl_xor_sync(FULL, pp, o);
    nx += __shfl_xor_sync(FULL, nx, o);
    ny += __shfl_xor_sync(FULL, ny, o);
  }
  __shared__ R rnum[2][PRIM_THREADS / 32];
  if (lane == 0) {
    red[0][w] = yy;
    red[1][w] = pp;
    rnum[0][w] = nx;
    rnum[1][w] = ny;
  }
  __syncthreads();
  if (tid == 0) {
    R a = 0, c = 0, ux = 0, uy = 0;
    for (int k = 0; k < nw; ++k) {
      a += red[0][k];
      c += red[1][k];
      ux += rnum[0][k];
      uy += rnum[1][k];
    }
    const R den = a + (R)P.reg[b] * c;
    go = den != (R)0;
    if (go) gam = Cx<T>::make(ux / den, uy / den);
    if (stepped) *stepped = go;
  }
  __syncthreads();
  if (!go) return;
  const T g = gam;
  if (span) {
    for (int q = tid; q < n_span; q += blockDim.x) col[span[q]] = cadd(col[span[q]], np_smul(g, y[span[q]]));
  } else {
    for (int n = tid; n < Nt; n += blockDim.x) col[n] = cadd(col[n], np_smul(g, y[n]));
  }
  for (int q = tid; q < n_rows; q += blockDim.x) {
    const int i = rows[q];
    coef[i] = cadd(coef[i], np_smul(g, phi[i]));
  }
  (void)red;
}

}  // namespace kz
