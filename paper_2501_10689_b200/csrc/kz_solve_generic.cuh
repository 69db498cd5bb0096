// Generic batched Kaczmarz solver: one CTA per system, one warp per
// right-hand side at a time, full solver state in a resumable global
// workspace.  Handles every scheme / stop mode / support shape the reference
// handles (arbitrary multi-segment supports); the fast paths in
// kz_solve_lockstep.cuh cover the contiguous-VR throughput configs.
//
// Reference semantics restated here (pkg/src/kaczprec/solvers.py):
//   residual_refresh :143-170   rk_step :173-188   select_row :205-237
//   aggregation_weights :248-254   ahk_step :257-309
//   orthogonal_block_step :312-332   InstanceRun.step :382-423
//   solve :460-507   solve_all :510-537   run_precoding :556-603
// and the FlopCounter charges of each primitive (metrics.py:25-41).
#pragma once

#include "kz_common.cuh"

namespace kz {

constexpr int GEN_WARPS = 8;  // warps per CTA of the generic kernel

// ---------------------------------------------------------------- workspace
struct GenLayout {
  size_t M, Q, R, Y, iters, noop, prev, flags, draws, flops, pool, poolcnt, checks, sys_t, sys_flags, total;
};

__host__ __device__ inline size_t kz_align(size_t x) { return (x + 255) & ~size_t(255); }

__host__ __device__ inline GenLayout gen_layout(int B, int K, int Nt, int dtype) {
  size_t cs = dtype == KZ_C128 ? 16 : 8;
  size_t nrhs = (size_t)B * K;
  GenLayout L;
  size_t o = 0;
  L.M = o;       o = kz_align(o + nrhs * Nt * cs);
  L.Q = o;       o = kz_align(o + nrhs * K * cs);
  L.R = o;       o = kz_align(o + nrhs * K * cs);
  L.Y = o;       o = kz_align(o + (size_t)B * GEN_WARPS * Nt * cs);
  L.iters = o;   o = kz_align(o + nrhs * 4);
  L.noop = o;    o = kz_align(o + nrhs * 4);
  L.prev = o;    o = kz_align(o + nrhs * 4);
  L.flags = o;   o = kz_align(o + nrhs * 4);
  L.draws = o;   o = kz_align(o + nrhs * 8);
  L.flops = o;   o = kz_align(o + nrhs * 8);
  L.pool = o;    o = kz_align(o + nrhs * K);
  L.poolcnt = o; o = kz_align(o + nrhs * 4);
  L.checks = o;  o = kz_align(o + nrhs * 4);
  L.sys_t = o;   o = kz_align(o + (size_t)B * 4);
  L.sys_flags = o; o = kz_align(o + (size_t)B * 4);
  L.total = o;
  return L;
}

// per-rhs flag bits
enum : uint32_t { F_DONE = 1, F_CONV = 2, F_PAUSED = 4, F_FINISHED = 8 };
// per-system flag bits
enum : uint32_t { S_CONV = 1, S_FINISHED = 2, S_PAUSED = 4 };

// ---------------------------------------------------------------- context
template <class T> struct Gen {
  kz_problem P;
  kz_stop S;
  kz_rng G;
  kz_out O;
  int scheme;
  char* ws;
  GenLayout L;

  __device__ __forceinline__ int K() const { return P.n_users; }
  __device__ __forceinline__ int Nt() const { return P.n_antennas; }
  __device__ __forceinline__ size_t rid(int b, int c) const { return (size_t)b * P.n_users + c; }
  __device__ __forceinline__ T* M(int b, int c) const { return (T*)(ws + L.M) + rid(b, c) * Nt(); }
  __device__ __forceinline__ T* Qv(int b, int c) const { return (T*)(ws + L.Q) + rid(b, c) * K(); }
  __device__ __forceinline__ T* Rv(int b, int c) const { return (T*)(ws + L.R) + rid(b, c) * K(); }
  __device__ __forceinline__ T* Y(int b, int w) const { return (T*)(ws + L.Y) + ((size_t)b * GEN_WARPS + w) * Nt(); }
  __device__ __forceinline__ int32_t& iters(int b, int c) const { return ((int32_t*)(ws + L.iters))[rid(b, c)]; }
  __device__ __forceinline__ int32_t& noop(int b, int c) const { return ((int32_t*)(ws + L.noop))[rid(b, c)]; }
  __device__ __forceinline__ int32_t& prev(int b, int c) const { return ((int32_t*)(ws + L.prev))[rid(b, c)]; }
  __device__ __forceinline__ uint32_t& flags(int b, int c) const { return ((uint32_t*)(ws + L.flags))[rid(b, c)]; }
  __device__ __forceinline__ int64_t& draws(int b, int c) const { return ((int64_t*)(ws + L.draws))[rid(b, c)]; }
  __device__ __forceinline__ int64_t& flops(int b, int c) const { return ((int64_t*)(ws + L.flops))[rid(b, c)]; }
  __device__ __forceinline__ uint8_t* pool(int b, int c) const { return (uint8_t*)(ws + L.pool) + rid(b, c) * K(); }
  __device__ __forceinline__ int32_t& poolcnt(int b, int c) const { return ((int32_t*)(ws + L.poolcnt))[rid(b, c)]; }
  __device__ __forceinline__ int32_t& checks(int b, int c) const { return ((int32_t*)(ws + L.checks))[rid(b, c)]; }
  __device__ __forceinline__ int32_t& sys_t(int b) const { return ((int32_t*)(ws + L.sys_t))[b]; }
  __device__ __forceinline__ uint32_t& sys_flags(int b) const { return ((uint32_t*)(ws + L.sys_flags))[b]; }

  __device__ __forceinline__ const T* H() const { return (const T*)P.heff; }
  __device__ __forceinline__ int support(int b, int i) const {
    size_t r = rid(b, i);
    return (int)(P.row_val_ptr[r + 1] - P.row_val_ptr[r]);
  }
  __device__ __forceinline__ double energy(int b, int i) const { return P.row_energy[rid(b, i)]; }

  __device__ __forceinline__ bool stochastic() const {
    return scheme == KZ_URK || scheme == KZ_SWOR_ERK || scheme == KZ_GRK || scheme == KZ_VR_OGRK;
  }
  __device__ __forceinline__ bool host_stream() const {
    return G.kind == KZ_RNG_HOST_UNIFORM || G.kind == KZ_RNG_HOST_INDEX;
  }
  __device__ __forceinline__ bool out_of_draws(int b, int c) const {
    return stochastic() && host_stream() && draws(b, c) >= G.stream_base + G.stream_len;
  }
  __device__ __forceinline__ double uniform(int b, int c) const {
    int64_t d = draws(b, c);
    if (G.kind == KZ_RNG_PHILOX) return philox_uniform(G.seed, (uint32_t)(b + G.system_base), (uint32_t)c, (uint64_t)d);
    return G.uniforms[rid(b, c) * G.stream_len + (d - G.stream_base)];
  }
  __device__ __forceinline__ int index_draw(int b, int c) const {
    return G.indices[rid(b, c) * G.stream_len + (draws(b, c) - G.stream_base)];
  }

  // ---------------------------------------------------------------- primitives
  // h_i^H m over the support of row i (warp-cooperative, result in every lane)
  __device__ T row_dot(int b, int i, const T* m, int lane) const {
    size_t r = rid(b, i);
    int s0 = P.row_seg_ptr[r], s1 = P.row_seg_ptr[r + 1];
    int64_t v = P.row_val_ptr[r];
    const T* h = H();
    T acc = czero<T>();
    for (int s = s0; s < s1; ++s) {
      int st = P.seg_start[s], ln = P.seg_len[s];
      for (int j = lane; j < ln; j += 32) acc = cfma_conj(h[v + j], m[st + j], acc);
      v += ln;
    }
    return warp_csum(acc);
  }
  // m[Gamma_i] += g * h_i  (numpy: col[idx] += gamma * eff_rows[i])
  __device__ void row_axpy(int b, int i, T g, T* m, int lane) const {
    size_t r = rid(b, i);
    int s0 = P.row_seg_ptr[r], s1 = P.row_seg_ptr[r + 1];
    int64_t v = P.row_val_ptr[r];
    const T* h = H();
    for (int s = s0; s < s1; ++s) {
      int st = P.seg_start[s], ln = P.seg_len[s];
      for (int j = lane; j < ln; j += 32) m[st + j] = cadd(m[st + j], cmul(g, h[v + j]));
      v += ln;
    }
    __syncwarp();
  }

  // dense-form residual of row i: -(h_i^H m) - reg q_i (+1 if i == rhs)  (solvers.py:149-153)
  __device__ T resid_dense(int b, int c, int i, const T* m, const T* q, int lane) const {
    T dot = row_dot(b, i, m, lane);
    double reg = P.reg[b];
    T rq = cscale(q[i], (typename Cx<T>::real)reg);
    T r = Cx<T>::make(-dot.x - rq.x, -dot.y - rq.y);
    if (i == c) r.x += (typename Cx<T>::real)1.0;
    return r;
  }
  // VR-form residual: target - dot - reg q_i  (solvers.py:166)
  __device__ T resid_vr(int b, int c, int i, const T* m, const T* q, int lane) const {
    T dot = row_dot(b, i, m, lane);
    double reg = P.reg[b];
    T rq = cscale(q[i], (typename Cx<T>::real)reg);
    typename Cx<T>::real tgt = i == c ? 1 : 0;
    return Cx<T>::make((tgt - dot.x) - rq.x, (0 - dot.y) - rq.y);
  }

  __device__ void refresh_all_dense(int b, int c, int lane) const {
    T* m = M(b, c);
    T* q = Qv(b, c);
    T* r = Rv(b, c);
    for (int i = 0; i < K(); ++i) {
      T v = resid_dense(b, c, i, m, q, lane);
      if (lane == 0) r[i] = v;
    }
    __syncwarp();
  }
  __device__ int64_t refresh_rows_vr(int b, int c, const int32_t* rows, int n, int lane) const {
    T* m = M(b, c);
    T* q = Qv(b, c);
    T* r = Rv(b, c);
    int64_t f = 0;
    for (int k = 0; k < n; ++k) {
      int i = rows[k];
      T v = resid_vr(b, c, i, m, q, lane);
      if (lane == 0) r[i] = v;
      f += 8 * (int64_t)support(b, i) + 4;
    }
    __syncwarp();
    return f;
  }
  // rk_step: project on row i with the stored residual (solvers.py:173-188)
  __device__ void rk_project(int b, int c, int i, int lane) const {
    T* r = Rv(b, c);
    T g = cdivr(r[i], energy(b, i));
    row_axpy(b, i, g, M(b, c), lane);
    if (lane == 0) {
      T* q = Qv(b, c);
      q[i] = cadd(q[i], g);
      r[i] = czero<T>();
    }
    __syncwarp();
  }

  // greedy-weighted pick (solvers.py:231-237); -1 when total == 0
  __device__ int pick_weighted(int b, int c, double* wbuf, double* cbuf, int lane, bool& drew) const {
    const T* r = Rv(b, c);
    int k = K();
    for (int i = lane; i < k; i += 32) wbuf[i] = np_abs2((double)r[i].x, (double)r[i].y);
    __syncwarp();
    double total = 0.0;
    if (lane == 0) total = np_pairwise_sum(wbuf, k);
    total = __shfl_sync(FULL, total, 0);
    drew = false;
    if (total == 0.0) return -1;
    for (int i = lane; i < k; i += 32) wbuf[i] = wbuf[i] / total;
    __syncwarp();
    if (lane == 0) {
      double acc = 0.0;
      for (int i = 0; i < k; ++i) {
        acc += wbuf[i];
        cbuf[i] = acc;
      }
    }
    __syncwarp();
    double last = cbuf[k - 1];
    double u = uniform(b, c);
    drew = true;
    for (int base = 0; base < k; base += 32) {
      int i = base + lane;
      bool hit = i < k && (cbuf[i] / last > u);
      unsigned bal = __ballot_sync(FULL, hit);
      if (bal) return base + __ffs(bal) - 1;
    }
    return k - 1;
  }
  // greedy-max pick (solvers.py:210-215); -1 when every score is zero
  __device__ int pick_max(int b, int c, int lane) const {
    const T* r = Rv(b, c);
    double best = -1.0;
    int bi = 0x7fffffff;
    bool any = false;
    for (int i = lane; i < K(); i += 32) {
      double s = np_abs2((double)r[i].x, (double)r[i].y) / energy(b, i);
      if (s != 0.0) any = true;
      if (s > best) { best = s; bi = i; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      double ob = __shfl_xor_sync(FULL, best, o);
      int oi = __shfl_xor_sync(FULL, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    any = __any_sync(FULL, any);
    return any ? bi : -1;
  }
  // energy-swor pick with an on-device pool (Philox mode); host streams pass indices
  __device__ int pick_swor_philox(int b, int c, int lane) const {
    uint8_t* pl = pool(b, c);
    int k = K();
    int i_sel = 0;
    if (lane == 0) {
      if (poolcnt(b, c) == 0) {
        for (int i = 0; i < k; ++i) pl[i] = 1;
        poolcnt(b, c) = k;
      }
      double tot = 0.0;
      for (int i = 0; i < k; ++i) if (pl[i]) tot += energy(b, i);
      double u = uniform(b, c) * tot, acc = 0.0;
      int last = -1;
      i_sel = -1;
      for (int i = 0; i < k; ++i) {
        if (!pl[i]) continue;
        last = i;
        acc += energy(b, i);
        if (acc > u) { i_sel = i; break; }
      }
      if (i_sel < 0) i_sel = last;
      pl[i_sel] = 0;
      poolcnt(b, c) -= 1;
    }
    return __shfl_sync(FULL, i_sel, 0);
  }

  __device__ void log_row(int b, int c, int it, int i) const {
    if (O.rows && it < O.rows_cap) O.rows[rid(b, c) * O.rows_cap + it] = i;
  }

  // |union of the supports of `rows`| (the span ahk_step charges, solvers.py:279-286): antennas marked in the
  // warp's y scratch, counted, cleared (ahk() zeroes y again before aggregating)
  __device__ int union_size(int b, const int32_t* rows, int nrows, int warp, int lane) const {
    T* y = Y(b, warp);
    const int nt = Nt();
    for (int n = lane; n < nt; n += 32) y[n] = czero<T>();
    __syncwarp();
    for (int k = 0; k < nrows; ++k) {
      size_t rr = rid(b, rows[k]);
      for (int s = P.row_seg_ptr[rr]; s < P.row_seg_ptr[rr + 1]; ++s) {
        const int st = P.seg_start[s], ln = P.seg_len[s];
        for (int j = lane; j < ln; j += 32) y[st + j] = Cx<T>::make(1, 0);
      }
      __syncwarp();
    }
    int cnt = 0;
    for (int n = lane; n < nt; n += 32) cnt += y[n].x != 0 ? 1 : 0;
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
    __syncwarp();
    return cnt;
  }

  // aggregated step over `rows` (solvers.py:257-309); dense==true mirrors use_vr=False.
  // phi is warp scratch [K].  Returns false on a no-op.
  __device__ bool ahk(int b, int c, const int32_t* rows, int nrows, bool dense, int span_size, T* phi,
                      int warp, int lane, int64_t& f) const {
    T* r = Rv(b, c);
    T* q = Qv(b, c);
    T* m = M(b, c);
    int nt = Nt();
    // weights phi_i = r_i / e_i (solvers.py:248-254)
    bool nz = false;
    for (int k = lane; k < nrows; k += 32) {
      int i = rows ? rows[k] : k;
      T p = cdivr(r[i], energy(b, i));
      phi[k] = p;
      if (p.x != 0 || p.y != 0) nz = true;
    }
    f += 2 * (int64_t)nrows;
    nz = __any_sync(FULL, nz);
    __syncwarp();
    if (nrows == 0 || !nz) return false;
    // num = vdot(phi, r)
    T num = czero<T>();
    for (int k = lane; k < nrows; k += 32) {
      int i = rows ? rows[k] : k;
      num = cfma_conj(phi[k], r[i], num);
    }
    num = warp_csum(num);
    f += 6 * (int64_t)nrows + 2 * (int64_t)max(nrows - 1, 0);
    // y = sum_i phi_i h_i, scattered in ascending row order
    T* y = Y(b, warp);
    for (int n = lane; n < nt; n += 32) y[n] = czero<T>();
    __syncwarp();
    for (int k = 0; k < nrows; ++k) {
      int i = rows ? rows[k] : k;
      size_t rr = rid(b, i);
      int s0 = P.row_seg_ptr[rr], s1 = P.row_seg_ptr[rr + 1];
      int64_t v = P.row_val_ptr[rr];
      T p = phi[k];
      for (int s = s0; s < s1; ++s) {
        int st = P.seg_start[s], ln = P.seg_len[s];
        for (int j = lane; j < ln; j += 32) y[st + j] = cadd(y[st + j], cmul(p, H()[v + j]));
        v += ln;
      }
      __syncwarp();
      if (!dense) f += 8 * (int64_t)support(b, i);
    }
    if (dense) f += 6 * (int64_t)nt * nrows + 2 * (int64_t)nt * max(nrows - 1, 0);
    // den = ||y||^2 + reg ||phi||^2
    double sy = 0.0, sp = 0.0;
    for (int n = lane; n < nt; n += 32) sy += np_abs2((double)y[n].x, (double)y[n].y);
    for (int k = lane; k < nrows; k += 32) sp += np_abs2((double)phi[k].x, (double)phi[k].y);
    sy = warp_sum(sy);
    sp = warp_sum(sp);
    double den = sy + P.reg[b] * sp;
    f += 4 * (int64_t)span_size + 3 * (int64_t)nrows + 2;
    if (den == 0.0) return false;
    double2 nd = to_d2(num);
    T g = from_d2<T>(make_double2(nd.x / den, nd.y / den));
    f += 2;
    for (int n = lane; n < nt; n += 32) m[n] = cadd(m[n], cmul(g, y[n]));
    f += 8 * (int64_t)span_size;
    for (int k = lane; k < nrows; k += 32) {
      int i = rows ? rows[k] : k;
      q[i] = cadd(q[i], cmul(g, phi[k]));
    }
    f += 8 * (int64_t)nrows;
    __syncwarp();
    return true;
  }

  // One scheme iteration of rhs c (InstanceRun.step, solvers.py:382-423).
  // Returns true if a step was taken (not already done).
  __device__ void step(int b, int c, double* wbuf, double* cbuf, T* phi, int warp, int lane) const {
    uint32_t fl = flags(b, c);
    if (fl & F_DONE) return;
    int k = K(), nt = Nt();
    int64_t f = 0;
    int it = iters(b, c);
    switch (scheme) {
      case KZ_URK:
      case KZ_SWOR_ERK: {
        int i;
        if (scheme == KZ_SWOR_ERK) f += (k - (int)(draws(b, c) % k)) + 2;
        if (G.kind == KZ_RNG_HOST_INDEX) i = index_draw(b, c);
        else if (scheme == KZ_URK) { i = (int)(uniform(b, c) * k); i = i >= k ? k - 1 : i; }
        else i = pick_swor_philox(b, c, lane);
        if (lane == 0) draws(b, c) += 1;
        // residual_refresh(rows=(i,), use_vr=False): target - dot - reg q
        T v = resid_vr(b, c, i, M(b, c), Qv(b, c), lane);
        if (lane == 0) Rv(b, c)[i] = v;
        __syncwarp();
        f += 8 * (int64_t)nt + 4;
        rk_project(b, c, i, lane);
        f += 2 + 8 * (int64_t)nt + 2;
        log_row(b, c, it, i);
        it += 1;
        break;
      }
      case KZ_GK:
      case KZ_GRK: {
        refresh_all_dense(b, c, lane);
        f += 6 * (int64_t)k * nt + 2 * (int64_t)k * (nt + 1) + 2 * (int64_t)k;
        int i;
        if (scheme == KZ_GK) {
          f += 4 * (int64_t)k;
          i = pick_max(b, c, lane);
        } else {
          f += 4 * (int64_t)k + 2;
          bool drew;
          i = pick_weighted(b, c, wbuf, cbuf, lane, drew);
          if (drew && lane == 0) draws(b, c) += 1;
        }
        if (i < 0) {
          fl |= F_DONE;
          break;
        }
        rk_project(b, c, i, lane);
        f += 2 + 8 * (int64_t)nt + 2;
        log_row(b, c, it, i);
        it += 1;
        break;
      }
      case KZ_VR_OGRK: {
        int pr = prev(b, c);
        if (pr >= 0) {
          size_t rr = rid(b, pr);
          int a0 = P.coupled_ptr[rr], a1 = P.coupled_ptr[rr + 1];
          f += refresh_rows_vr(b, c, P.coupled_idx + a0, a1 - a0, lane);
        }
        f += 4 * (int64_t)k + 2;
        bool drew;
        int i = pick_weighted(b, c, wbuf, cbuf, lane, drew);
        if (drew && lane == 0) draws(b, c) += 1;
        if (i < 0) {
          fl |= F_DONE;
          break;
        }
        rk_project(b, c, i, lane);
        f += 2 + 8 * (int64_t)support(b, i) + 2;
        if (lane == 0) prev(b, c) = i;
        log_row(b, c, it, i);
        it += 1;
        break;
      }
      case KZ_AHK: {
        refresh_all_dense(b, c, lane);
        f += 6 * (int64_t)k * nt + 2 * (int64_t)k * (nt + 1) + 2 * (int64_t)k;
        bool ok = ahk(b, c, nullptr, k, true, nt, phi, warp, lane, f);
        if (!ok) {
          if (lane == 0) noop(b, c) += 1;
          fl |= F_DONE;
          break;
        }
        it += 1;
        break;
      }
      case KZ_VR_OAHK: {
        int o0 = P.orth_ptr[b], o1 = P.orth_ptr[b + 1];
        const int32_t* orows = P.orth_idx + o0;
        f += refresh_rows_vr(b, c, orows, o1 - o0, lane);
        for (int kk = 0; kk < o1 - o0; ++kk) {  // disjoint supports: order-independent
          int i = orows[kk];
          rk_project(b, c, i, lane);
          f += 2 + 8 * (int64_t)support(b, i) + 2;
        }
        int n0 = P.non_ptr[b], n1 = P.non_ptr[b + 1];
        if (n1 > n0) {
          const int32_t* nrows = P.non_idx + n0;
          f += refresh_rows_vr(b, c, nrows, n1 - n0, lane);
          bool ok = ahk(b, c, nrows, n1 - n0, false, P.non_union_size[b], phi, warp, lane, f);
          if (!ok && lane == 0) noop(b, c) += 1;
        }
        it += 1;
        break;
      }
      case KZ_VR_OAHK_G: {  // oracle/grouped.py GroupedRun.step
        for (int gi = P.ogrp_sys[b]; gi < P.ogrp_sys[b + 1]; ++gi) {
          const int o0 = P.ogrp_ptr[gi], o1 = P.ogrp_ptr[gi + 1];
          const int32_t* orows = P.orth_idx + o0;
          f += refresh_rows_vr(b, c, orows, o1 - o0, lane);
          for (int kk = 0; kk < o1 - o0; ++kk) {  // one group: disjoint supports, order-independent
            const int i = orows[kk];
            rk_project(b, c, i, lane);
            f += 2 + 8 * (int64_t)support(b, i) + 2;
          }
        }
        const int n0 = P.non_ptr[b], n1 = P.non_ptr[b + 1], cap = P.agg_cap;
        for (int s0 = n0; s0 < n1; s0 += cap) {  // consecutive ascending blocks of at most agg_cap rows
          const int nb = min(cap, n1 - s0);
          const int32_t* brows = P.non_idx + s0;
          f += refresh_rows_vr(b, c, brows, nb, lane);
          const int span = union_size(b, brows, nb, warp, lane);
          bool ok = ahk(b, c, brows, nb, false, span, phi, warp, lane, f);
          if (!ok && lane == 0) noop(b, c) += 1;
        }
        it += 1;
        break;
      }
    }
    if (lane == 0) {
      iters(b, c) = it;
      flops(b, c) += f;
      flags(b, c) = fl;
    }
    __syncwarp();
  }

  // ||e_c - H^H m - reg q||_2 with fresh residuals (solvers.py:453-457), not stored
  __device__ double true_resid_sq(int b, int c, int lane) const {
    const T* m = M(b, c);
    const T* q = Qv(b, c);
    double s = 0.0;
    for (int i = 0; i < K(); ++i) {
      T v = resid_dense(b, c, i, m, q, lane);
      s += (double)v.x * v.x + (double)v.y * v.y;
    }
    return s;  // identical in every lane
  }
};

// block-wide double sum (all threads participate; result broadcast)
__device__ inline double block_sum(double v, double* red) {
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

template <class T>
__global__ void __launch_bounds__(GEN_WARPS * 32) kz_generic_kernel(Gen<T> g, int resume) {
  extern __shared__ double smem[];
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int K = g.K(), Nt = g.Nt();
  double* wbuf = smem + (size_t)warp * 2 * K;
  double* cbuf = wbuf + K;
  T* phi = (T*)(smem + (size_t)nw * 2 * K) + (size_t)warp * K;
  __shared__ double red[32];
  __shared__ int s_flag;

  // ---- initial state (SolverState.initial, solvers.py:129-136)
  if (!resume) {
    for (int c = warp; c < K; c += nw) {
      T* m = g.M(b, c);
      for (int n = lane; n < Nt; n += 32) m[n] = czero<T>();
      T* q = g.Qv(b, c);
      T* r = g.Rv(b, c);
      for (int i = lane; i < K; i += 32) {
        q[i] = czero<T>();
        r[i] = i == c ? Cx<T>::make(1, 0) : czero<T>();
        g.pool(b, c)[i] = 0;
      }
      if (lane == 0) {
        g.iters(b, c) = 0;
        g.noop(b, c) = 0;
        g.prev(b, c) = -1;
        bool masked = g.S.rhs_mask && !g.S.rhs_mask[g.rid(b, c)];
        g.flags(b, c) = masked ? (F_DONE | F_FINISHED) : 0;
        g.checks(b, c) = 0;
        g.draws(b, c) = 0;
        g.flops(b, c) = 0;
        g.poolcnt(b, c) = 0;
      }
    }
    if (threadIdx.x == 0) {
      g.sys_t(b) = 0;
      g.sys_flags(b) = 0;
    }
    __syncthreads();
  }

  if (g.S.mode == KZ_STOP_LOCKSTEP) {
    // ---- run_precoding lockstep driver (solvers.py:583-603)
    if (g.sys_flags(b) & S_FINISHED) return;
    const bool need_nmse = g.S.epsilon > 0.0 || g.O.nmse_trace;
    const double* fref = g.S.f_ref ? g.S.f_ref + (size_t)b * Nt * K * 2 : nullptr;
    double fref_norm = 0.0;
    if (need_nmse && fref) {
      double s = 0.0;
      for (size_t e = threadIdx.x; e < (size_t)Nt * K; e += blockDim.x) s += fref[2 * e] * fref[2 * e] + fref[2 * e + 1] * fref[2 * e + 1];
      fref_norm = sqrt(block_sum(s, red));
    }
    int cap = g.S.max_iters;
    int t = g.sys_t(b);
    while (true) {
      // pause before an outer iteration that would need draws we do not have
      if (threadIdx.x == 0) s_flag = 0;
      __syncthreads();
      for (int c = warp; c < K; c += nw)
        if (!(g.flags(b, c) & F_DONE) && g.out_of_draws(b, c) && lane == 0) s_flag = 1;
      __syncthreads();
      if (s_flag) {
        if (threadIdx.x == 0) {
          g.sys_t(b) = t;
          g.sys_flags(b) |= S_PAUSED;
        }
        for (int c = warp; c < K; c += nw)
          if (lane == 0 && g.O.paused) g.O.paused[g.rid(b, c)] = 1;
        break;
      }
      t += 1;
      for (int c = warp; c < K; c += nw) g.step(b, c, wbuf, cbuf, phi, warp, lane);
      __syncthreads();
      bool conv = false;
      if (need_nmse) {
        double s1 = 0.0;
        for (int c = warp; c < K; c += nw) {
          const T* m = g.M(b, c);
          for (int n = lane; n < Nt; n += 32) s1 += (double)m[n].x * m[n].x + (double)m[n].y * m[n].y;
        }
        double mn = sqrt(block_sum(s1, red));
        double s2 = 0.0;
        for (int c = warp; c < K; c += nw) {
          const T* m = g.M(b, c);
          for (int n = lane; n < Nt; n += 32) {
            double mr = m[n].x, mi = m[n].y;
            if (mn > 0.0) { mr /= mn; mi /= mn; }
            double dr = fref[2 * ((size_t)n * K + c)] - mr, di = fref[2 * ((size_t)n * K + c) + 1] - mi;
            s2 += dr * dr + di * di;
          }
        }
        double err = sqrt(block_sum(s2, red)) / fref_norm;
        if (g.O.nmse_trace && t - 1 < g.O.trace_cap && threadIdx.x == 0) g.O.nmse_trace[(size_t)b * g.O.trace_cap + t - 1] = err;
        conv = err < g.S.epsilon;
      }
      if (g.O.resid_trace && t - 1 < g.O.trace_cap) {
        double s = 0.0;
        for (int c = warp; c < K; c += nw) s += g.true_resid_sq(b, c, lane) * (lane == 0 ? 1.0 : 0.0);
        double tot = block_sum(s, red);
        if (threadIdx.x == 0) g.O.resid_trace[(size_t)b * g.O.trace_cap + t - 1] = sqrt(tot);
      }
      if (g.O.flops_trace && t - 1 < g.O.trace_cap && threadIdx.x == 0) {
        int64_t fs = 0;
        for (int c = 0; c < K; ++c) fs += g.flops(b, c);
        g.O.flops_trace[(size_t)b * g.O.trace_cap + t - 1] = fs;
      }
      if (threadIdx.x == 0) s_flag = 1;
      __syncthreads();
      for (int c = warp; c < K; c += nw)
        if (lane == 0 && !(g.flags(b, c) & F_DONE)) s_flag = 0;
      __syncthreads();
      bool all_done = s_flag;
      __syncthreads();
      if (conv || t >= cap || all_done) {
        if (threadIdx.x == 0) {
          g.sys_t(b) = t;
          g.sys_flags(b) = (conv ? S_CONV : 0) | S_FINISHED;
        }
        break;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (g.O.n_outer) g.O.n_outer[b] = g.sys_t(b);
      if (g.O.sys_converged) g.O.sys_converged[b] = (g.sys_flags(b) & S_CONV) ? 1 : 0;
    }
  } else {
    // ---- solve / solve_all: independent per-rhs loops (solvers.py:480-503)
    const int cap = g.S.max_iters;
    const int every = g.S.check_every;
    for (int c = warp; c < K; c += nw) {
      uint32_t fl = g.flags(b, c);
      if (fl & F_FINISHED) continue;
      const double* vref = g.S.v_ref ? g.S.v_ref + (size_t)b * K * K * 2 : nullptr;
      double ref_norm = 0.0;
      if (g.S.mode == KZ_STOP_ORACLE) {
        double s = 0.0;
        for (int i = lane; i < K; i += 32) {
          double a = vref[2 * ((size_t)i * K + c)], bb = vref[2 * ((size_t)i * K + c) + 1];
          s += a * a + bb * bb;
        }
        ref_norm = sqrt(warp_sum(s));
      }
      while (true) {
        if (g.out_of_draws(b, c) && !(g.flags(b, c) & F_DONE)) {
          if (lane == 0) {
            g.flags(b, c) |= F_PAUSED;
            if (g.O.paused) g.O.paused[g.rid(b, c)] = 1;
          }
          break;
        }
        g.step(b, c, wbuf, cbuf, phi, warp, lane);
        fl = g.flags(b, c);
        int it = g.iters(b, c);
        bool done = fl & F_DONE;
        bool conv = false;
        if (it % every == 0 || done) {
          // _true_residual_norm is evaluated at every check in both modes (solvers.py:484-486)
          double rn = sqrt(g.true_resid_sq(b, c, lane));
          double err = 0.0;
          if (g.S.mode == KZ_STOP_RESIDUAL) {
            conv = rn <= g.S.epsilon;
          } else {
            const T* q = g.Qv(b, c);
            double s = 0.0;
            for (int i = lane; i < K; i += 32) {
              double a = (double)q[i].x - vref[2 * ((size_t)i * K + c)];
              double bb = (double)q[i].y - vref[2 * ((size_t)i * K + c) + 1];
              s += a * a + bb * bb;
            }
            err = sqrt(warp_sum(s)) / ref_norm;
            conv = err < g.S.epsilon;
          }
          if (lane == 0) {
            int ck = g.checks(b, c);
            if (ck < g.O.trace_cap) {
              size_t o = g.rid(b, c) * g.O.trace_cap + ck;
              if (g.O.resid_trace) g.O.resid_trace[o] = rn;
              if (g.O.nmse_trace) g.O.nmse_trace[o] = err;
              if (g.O.flops_trace) g.O.flops_trace[o] = g.flops(b, c);
            }
            g.checks(b, c) = ck + 1;
          }
        }
        if (conv || done) {
          if (lane == 0) g.flags(b, c) = fl | F_CONV | F_FINISHED;
          break;
        }
        if (it >= cap) {
          if (lane == 0) g.flags(b, c) = fl | F_FINISHED;
          break;
        }
      }
      __syncwarp();
    }
    __syncthreads();
  }

  // ---- outputs: v[b][i][c] = coef_i of rhs c, per-rhs counters, optional iterates
  for (int c = warp; c < K; c += nw) {
    if (g.O.iterates) {
      const T* m = g.M(b, c);
      T* mo = (T*)g.O.iterates + g.rid(b, c) * Nt;
      for (int n = lane; n < Nt; n += 32) mo[n] = m[n];
    }
    const T* q = g.Qv(b, c);
    T* v = (T*)g.O.v;
    for (int i = lane; i < K; i += 32) v[((size_t)b * K + i) * K + c] = q[i];
    if (lane == 0) {
      size_t r = g.rid(b, c);
      uint32_t fl = g.flags(b, c);
      if (g.O.iters) g.O.iters[r] = g.iters(b, c);
      if (g.O.converged) g.O.converged[r] = (fl & F_CONV) ? 1 : 0;
      if (g.O.done) g.O.done[r] = (fl & F_DONE) ? 1 : 0;
      if (g.O.noop_steps) g.O.noop_steps[r] = g.noop(b, c);
      if (g.O.n_checks) g.O.n_checks[r] = g.checks(b, c);
      if (g.O.flops) g.O.flops[r] = g.flops(b, c);
    }
  }
}

}  // namespace kz
