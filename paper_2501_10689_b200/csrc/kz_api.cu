// C-ABI entry points of libkaczmarz_b200.so (see include/kaczmarz_b200.h).
//
// Validation mirrors the reference's ValueError conditions where they apply
// to a packed batch (solvers.py:48-52, 76-92, 351-352, 444-450; rzf.py:51-59).
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>

#include "kz_common.cuh"
#include "kz_dense.cuh"
#include "kz_solve_generic.cuh"
#include "kz_solve_lockstep.cuh"
#include "kz_solve_cluster.cuh"
#include "kz_channel.cuh"
#include "kz_primitives.cuh"

namespace {

thread_local std::string g_err;
thread_local int32_t g_launches = 0;

__attribute__((format(printf, 2, 3))) int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_check(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_err = std::string(where) + ": " + cudaGetErrorString(e);
    return KZ_ERR_CUDA;
  }
  return KZ_OK;
}

int check_problem(const kz_problem* p) {
  if (!p) return fail(KZ_ERR_INVALID, "null problem");
  if (p->n_systems < 0) return fail(KZ_ERR_INVALID, "n_systems must be >= 0 (got %d)", (int)p->n_systems);
  if (p->n_users < 1) return fail(KZ_ERR_INVALID, "need at least one user (got %d)", (int)p->n_users);
  if (p->n_antennas < 1) return fail(KZ_ERR_INVALID, "need at least one antenna (got %d)", (int)p->n_antennas);
  if (p->dtype != KZ_C128 && p->dtype != KZ_C64) return fail(KZ_ERR_INVALID, "unknown dtype %d", (int)p->dtype);
  if (p->n_systems == 0) return KZ_OK;
  if (!p->row_seg_ptr || !p->seg_start || !p->seg_len || !p->row_val_ptr || !p->heff || !p->row_energy || !p->reg)
    return fail(KZ_ERR_INVALID, "problem arrays must be non-null");
  return KZ_OK;
}

}  // namespace

using namespace kz;

extern "C" {

int32_t kz_abi_version(void) { return KZ_ABI_VERSION; }
const char* kz_last_error(void) { return g_err.c_str(); }
int32_t kz_last_launch_count(void) { return g_launches; }
int32_t kz_last_tma_staging(void) { return g_last_tma; }

size_t kz_solve_workspace_bytes(const kz_problem* prob, const kz_stop* stop) {
  (void)stop;
  if (!prob) return 0;
  size_t gen = gen_layout(prob->n_systems, prob->n_users, prob->n_antennas, prob->dtype).total;
  return gen > ls_extra_ws(*prob) ? gen : ls_extra_ws(*prob);
}

size_t kz_solve_workspace_bytes_for(const kz_problem* prob, int32_t scheme, const kz_stop* stop, const kz_rng* rng,
                                    const kz_out* out) {
  if (!prob || !stop || !rng || !out) return 0;
  if (prob->n_systems == 0) return 0;
  // ask the fast-path dispatchers which kernel kz_solve(resume = 0) would take, without launching anything
  int32_t dummy = 0;
  g_dry_launch = true;
  int fast = lockstep_try_launch(*prob, scheme, *stop, *rng, *out, 0, nullptr, ~size_t(0), nullptr, &dummy);
  bool clu = false;
  if (fast != 1) {
    fast = cluster_try_launch(*prob, scheme, *stop, *rng, *out, 0, nullptr, ~size_t(0), nullptr, &dummy);
    clu = fast == 1;
  }
  g_dry_launch = false;
  cudaGetLastError();  // eligibility probes (attributes, occupancy) leave no sticky error behind
  // the on-chip kernels keep only the stop iterations in HBM (the streamed cluster variant also its padded H_eff)
  if (fast == 1) return clu ? g_cluster_dry_ws : ls_extra_ws(*prob);
  return gen_layout(prob->n_systems, prob->n_users, prob->n_antennas, prob->dtype).total;
}

size_t kz_solve_resid_offset(const kz_problem* prob) {
  if (!prob) return 0;
  return gen_layout(prob->n_systems, prob->n_users, prob->n_antennas, prob->dtype).R;
}

int kz_solve(const kz_problem* prob, int32_t scheme, const kz_stop* stop, const kz_rng* rng, kz_out* out,
             void* workspace, size_t workspace_bytes, int32_t resume, void* stream) {
  g_launches = 0;
  g_last_tma = 0;
  int st = check_problem(prob);
  if (st) return st;
  if (scheme < KZ_URK || scheme > KZ_VR_OAHK_G) return fail(KZ_ERR_INVALID, "unknown scheme %d", (int)scheme);
  if (!stop || !rng || !out) return fail(KZ_ERR_INVALID, "null stop/rng/out");
  if (stop->mode < KZ_STOP_LOCKSTEP || stop->mode > KZ_STOP_ORACLE)
    return fail(KZ_ERR_INVALID, "unknown stopping mode %d", (int)stop->mode);
  if (stop->max_iters < 1) return fail(KZ_ERR_INVALID, "max_iters must be >= 1 (got %d)", (int)stop->max_iters);
  if (stop->check_every < 1) return fail(KZ_ERR_INVALID, "check_every must be >= 1");
  if (stop->mode == KZ_STOP_LOCKSTEP) {
    if (stop->epsilon < 0.0) return fail(KZ_ERR_INVALID, "epsilon must be >= 0 in lockstep mode");
    if ((stop->epsilon > 0.0 || out->nmse_trace) && !stop->f_ref)
      return fail(KZ_ERR_INVALID, "lockstep NMSE stopping needs f_ref");
  } else {
    if (!(stop->epsilon > 0.0)) return fail(KZ_ERR_INVALID, "epsilon must be positive");
    if (stop->mode == KZ_STOP_ORACLE && !stop->v_ref)
      return fail(KZ_ERR_INVALID, "oracle stopping needs the direct-solver reference");
  }
  const bool stochastic = scheme == KZ_URK || scheme == KZ_SWOR_ERK || scheme == KZ_GRK || scheme == KZ_VR_OGRK;
  if (stochastic) {
    bool idx_scheme = scheme == KZ_URK || scheme == KZ_SWOR_ERK;
    if (rng->kind == KZ_RNG_NONE) return fail(KZ_ERR_INVALID, "scheme draws rows at random; pass an rng");
    if (rng->kind == KZ_RNG_HOST_UNIFORM && (idx_scheme || !rng->uniforms))
      return fail(KZ_ERR_INVALID, "host uniform streams are for grk / vr-ogrk");
    if (rng->kind == KZ_RNG_HOST_INDEX && (!idx_scheme || !rng->indices))
      return fail(KZ_ERR_INVALID, "host index streams are for urk / swor-erk");
    if ((rng->kind == KZ_RNG_HOST_UNIFORM || rng->kind == KZ_RNG_HOST_INDEX) && rng->stream_len < 0)
      return fail(KZ_ERR_INVALID, "negative stream_len");
  }
  if ((scheme == KZ_VR_OGRK) && (!prob->coupled_ptr || !prob->coupled_idx))
    return fail(KZ_ERR_INVALID, "vr-ogrk needs the coupled sets");
  if ((scheme == KZ_VR_OAHK) && (!prob->orth_ptr || !prob->non_ptr || !prob->non_union_size))
    return fail(KZ_ERR_INVALID, "vr-oahk needs the orthogonal / non-orthogonal partition");
  if (scheme == KZ_VR_OAHK_G && (!prob->orth_ptr || !prob->non_ptr || !prob->ogrp_sys || !prob->ogrp_ptr))
    return fail(KZ_ERR_INVALID, "vr-oahk-g needs the orthogonal groups and the non-orthogonal rows");
  if (scheme == KZ_VR_OAHK_G && prob->agg_cap < 1)
    return fail(KZ_ERR_INVALID, "vr-oahk-g needs agg_cap >= 1 (got %d)", (int)prob->agg_cap);
  if (!out->v) return fail(KZ_ERR_INVALID, "out->v must be non-null");
  if (prob->n_systems == 0) return KZ_OK;
  if (!workspace) workspace_bytes = 0;

  cudaStream_t s = (cudaStream_t)stream;
  const int K = prob->n_users;
  // fast path: fixed-T lockstep over contiguous supports (kz_solve_lockstep.cuh)
  int fast = lockstep_try_launch(*prob, scheme, *stop, *rng, *out, resume, (char*)workspace, workspace_bytes, s,
                                 &g_launches);
  if (fast == 1) return cuda_check("kz_solve(lockstep)");
  if (fast < 0) return fail(KZ_ERR_CUDA, "lockstep launch failed");
  // large arrays / residual tolerance: one thread-block cluster per (system, 16 rhs) (kz_solve_cluster.cuh)
  fast = cluster_try_launch(*prob, scheme, *stop, *rng, *out, resume, (char*)workspace, workspace_bytes, s,
                            &g_launches);
  if (fast == 1) return cuda_check("kz_solve(cluster)");
  if (fast < 0) return fail(KZ_ERR_CUDA, "cluster launch failed");

  // generic kernel: the per-rhs state (iterates, residuals, counters) lives in the workspace
  const size_t need = gen_layout(prob->n_systems, K, prob->n_antennas, prob->dtype).total;
  if (!workspace || workspace_bytes < need)
    return fail(KZ_ERR_WORKSPACE, "workspace too small: need %lld bytes", (long long)need);
  const int nw = GEN_WARPS;
  size_t cs = prob->dtype == KZ_C128 ? 16 : 8;
  size_t smem = (size_t)nw * 2 * K * sizeof(double) + (size_t)nw * K * cs;
  GenLayout L = gen_layout(prob->n_systems, K, prob->n_antennas, prob->dtype);
  if (prob->dtype == KZ_C128) {
    Gen<double2> g{*prob, *stop, *rng, *out, scheme, (char*)workspace, L};
    cudaFuncSetAttribute(kz_generic_kernel<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kz_generic_kernel<double2><<<prob->n_systems, nw * 32, smem, s>>>(g, resume);
  } else {
    Gen<float2> g{*prob, *stop, *rng, *out, scheme, (char*)workspace, L};
    cudaFuncSetAttribute(kz_generic_kernel<float2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kz_generic_kernel<float2><<<prob->n_systems, nw * 32, smem, s>>>(g, resume);
  }
  g_launches = 1;
  return cuda_check("kz_solve(generic)");
}

// batched Gram on the FP64 tensor cores (kz_gram_tc_kernel): contiguous supports, K <= 256
static bool gram_tc_ok(const kz_problem* prob) {
  static const bool off = getenv("KZ_GRAM_TC") && atoi(getenv("KZ_GRAM_TC")) == 0;
  return !off && (prob->flags & KZ_PROBLEM_CONTIGUOUS) && prob->n_users <= GRAM_TC_KMAX;
}
static void launch_gram_tc(const kz_problem* prob, double2* out, size_t sys_stride, int add_reg, cudaStream_t s) {
  if (prob->dtype == KZ_C128)
    kz_gram_tc_kernel<double2><<<prob->n_systems, GRAM_TC_THREADS, 0, s>>>(*prob, out, sys_stride, add_reg);
  else
    kz_gram_tc_kernel<float2><<<prob->n_systems, GRAM_TC_THREADS, 0, s>>>(*prob, out, sys_stride, add_reg);
}

// the blocked Gauss-Jordan kernel inverts in place in v_out; only the legacy kernel needs a workspace
static bool rzf_uses_gj(const kz_problem* prob) {
  int dev = 0, maxsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return getenv("KZ_RZF_LEGACY") == nullptr && maxsm > 0 && rzf_smem(prob->n_users) <= (size_t)maxsm;
}

size_t kz_rzf_workspace_bytes(const kz_problem* prob) {
  if (!prob) return 0;
  if (rzf_uses_gj(prob)) return 0;
  return kz_align((size_t)prob->n_systems * 2 * prob->n_users * prob->n_users * sizeof(double2));
}

int kz_rzf(const kz_problem* prob, double* v_out, double* f_out, double* beta_out, uint8_t* pd_ok, void* workspace,
           size_t workspace_bytes, void* stream) {
  g_launches = 0;
  int st = check_problem(prob);
  if (st) return st;
  if (!v_out) return fail(KZ_ERR_INVALID, "v_out must be non-null");
  if (prob->n_systems == 0) return KZ_OK;
  size_t need = kz_rzf_workspace_bytes(prob);
  if (need && (!workspace || workspace_bytes < need))
    return fail(KZ_ERR_WORKSPACE, "workspace too small: need %lld bytes", (long long)need);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t smem = rzf_smem(prob->n_users);
  if (rzf_uses_gj(prob)) {  // KZ_RZF_LEGACY=1: A/B switch to the unblocked Cholesky kernel
    const int nb = rzf_nb(prob->n_users);
    const int nthr = prob->n_users <= 96 ? 256 : RZF_THREADS;  // small Grams: fewer threads, cheaper barriers
    // the Gram on the FP64 tensor cores (contiguous supports; KZ_GRAM_TC=0: the CUDA-core pair sums)
    const int tc = gram_tc_ok(prob) ? 1 : 0;
    if (tc) launch_gram_tc(prob, (double2*)v_out, (size_t)prob->n_users * prob->n_users, 1, s);
    if (prob->dtype == KZ_C128) {
      cudaFuncSetAttribute(kz_rzf_gj_kernel<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kz_rzf_gj_kernel<double2><<<prob->n_systems, nthr, smem, s>>>(*prob, v_out, f_out, beta_out, pd_ok, nb, tc);
    } else {
      cudaFuncSetAttribute(kz_rzf_gj_kernel<float2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kz_rzf_gj_kernel<float2><<<prob->n_systems, nthr, smem, s>>>(*prob, v_out, f_out, beta_out, pd_ok, nb, tc);
    }
    g_launches = 1 + tc;
    return cuda_check("kz_rzf");
  } else if (prob->dtype == KZ_C128) {
    kz_rzf_kernel<double2><<<prob->n_systems, DENSE_THREADS, 0, s>>>(*prob, v_out, f_out, beta_out, pd_ok, (double2*)workspace);
  } else {
    kz_rzf_kernel<float2><<<prob->n_systems, DENSE_THREADS, 0, s>>>(*prob, v_out, f_out, beta_out, pd_ok, (double2*)workspace);
  }
  g_launches = 1;
  return cuda_check("kz_rzf");
}

// Gram-form epilogue for large K (contiguous VRs, F not requested): G0 and G0 V per system
static bool epilogue_gram_path(const kz_problem* prob) {
  static const int kmin = getenv("KZ_EPILOGUE_GRAM_KMIN") ? atoi(getenv("KZ_EPILOGUE_GRAM_KMIN")) : 32;
  return (prob->flags & KZ_PROBLEM_CONTIGUOUS) && prob->n_users >= kmin && getenv("KZ_EPILOGUE_ANTENNA") == nullptr;
}

int32_t kz_epilogue_uses_gram(const kz_problem* prob, int32_t want_f) {
  return prob && epilogue_gram_path(prob) && !want_f ? 1 : 0;
}

size_t kz_epilogue_workspace_bytes(const kz_problem* prob) {
  if (!prob) return 0;
  size_t gram = (size_t)prob->n_systems * prob->n_users * prob->n_users * sizeof(double2) *
                (epilogue_gram_path(prob) ? 2 : 1);
  size_t fbuf = (size_t)prob->n_systems * prob->n_antennas * prob->n_users * (prob->dtype == KZ_C128 ? 16 : 8);
  return kz_align(gram > fbuf ? gram : fbuf);
}

int kz_epilogue(const kz_problem* prob, const void* v, void* f_out, const double* v_ref, const double* beta_ref,
                const double* snr_linear, double* beta_out, double* nmse_out, double* rates_out, double* sum_rate_out,
                void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  int st = check_problem(prob);
  if (st) return st;
  if (!v) return fail(KZ_ERR_INVALID, "v must be non-null");
  if (v_ref && !beta_ref) return fail(KZ_ERR_INVALID, "v_ref needs beta_ref");
  if (prob->n_systems == 0) return KZ_OK;
  const bool gram_path = epilogue_gram_path(prob) && !f_out;
  size_t need = (snr_linear || gram_path) ? kz_epilogue_workspace_bytes(prob) : 0;
  if (need && (!workspace || workspace_bytes < need))
    return fail(KZ_ERR_WORKSPACE, "workspace too small: need %lld bytes", (long long)need);
  cudaStream_t s = (cudaStream_t)stream;
  if (gram_path) {
    const size_t smem = epilogue_gram_smem();
    kz_problem pr = *prob;  // G0 on the tensor cores unless the caller's workspace already holds it
    int tc = 0;
    if (!(pr.flags & KZ_PROBLEM_GRAM_CACHED) && gram_tc_ok(prob)) {
      launch_gram_tc(prob, (double2*)workspace, 2 * (size_t)prob->n_users * prob->n_users, 0, s);
      pr.flags |= KZ_PROBLEM_GRAM_CACHED;
      tc = 1;
    }
    prob = &pr;
    if (prob->dtype == KZ_C128) {
      cudaFuncSetAttribute(kz_epilogue_gram_kernel<double2, double2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      kz_epilogue_gram_kernel<double2, double2><<<prob->n_systems, EPG_THREADS, smem, s>>>(
          *prob, (const double2*)v, v_ref, beta_ref, snr_linear, beta_out, nmse_out, rates_out, sum_rate_out,
          (double2*)workspace);
    } else {
      cudaFuncSetAttribute(kz_epilogue_gram_kernel<float2, float2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      kz_epilogue_gram_kernel<float2, float2><<<prob->n_systems, EPG_THREADS, smem, s>>>(
          *prob, (const float2*)v, v_ref, beta_ref, snr_linear, beta_out, nmse_out, rates_out, sum_rate_out,
          (double2*)workspace);
    }
    g_launches = 1 + tc;
    return cuda_check("kz_epilogue(gram)");
  }
  if (prob->flags & KZ_PROBLEM_CONTIGUOUS) {
    size_t smem = epilogue_contig_smem(prob->n_users);
    if (prob->dtype == KZ_C128)
      kz_epilogue_contig_kernel<double2><<<prob->n_systems, DENSE_THREADS, smem, s>>>(
          *prob, (const double2*)v, (double2*)f_out, v_ref, beta_ref, snr_linear, beta_out, nmse_out, rates_out,
          sum_rate_out, (double2*)workspace);
    else
      kz_epilogue_contig_kernel<float2><<<prob->n_systems, DENSE_THREADS, smem, s>>>(
          *prob, (const float2*)v, (float2*)f_out, v_ref, beta_ref, snr_linear, beta_out, nmse_out, rates_out,
          sum_rate_out, (float2*)workspace);
    g_launches = 1;
    return cuda_check("kz_epilogue(contiguous)");
  }
  if (prob->dtype == KZ_C128)
    kz_epilogue_kernel<double2><<<prob->n_systems, DENSE_THREADS, 0, s>>>(
        *prob, (const double2*)v, (double2*)f_out, v_ref, beta_ref, snr_linear, beta_out, nmse_out, rates_out,
        sum_rate_out, (double2*)workspace);
  else
    kz_epilogue_kernel<float2><<<prob->n_systems, DENSE_THREADS, 0, s>>>(
        *prob, (const float2*)v, (float2*)f_out, v_ref, beta_ref, snr_linear, beta_out, nmse_out, rates_out,
        sum_rate_out, (double2*)workspace);
  g_launches = 1;
  return cuda_check("kz_epilogue");
}

}  // extern "C"

// ------------------------------------------------------------------ on-device input preparation
static int check_drop(const kz_drop* d) {
  if (!d) return fail(KZ_ERR_INVALID, "drop is null");
  if (d->n_systems < 0 || d->n_users < 1 || d->n_antennas < 1)
    return fail(KZ_ERR_INVALID, "bad drop shape: B=%d K=%d Nt=%d", d->n_systems, d->n_users, d->n_antennas);
  if (d->dtype != KZ_C128 && d->dtype != KZ_C64) return fail(KZ_ERR_INVALID, "bad dtype %d", d->dtype);
  if (d->n_systems && (!d->wavelength || !d->r0 || !d->theta || !d->vr_start || !d->vr_len || !d->reg))
    return fail(KZ_ERR_INVALID, "drop arrays must be non-null");
  if (!(d->element_spacing > 0.0)) return fail(KZ_ERR_INVALID, "element_spacing must be positive");
  return KZ_OK;
}

extern "C" {

int kz_channel_synth(const kz_drop* drop, const int64_t* row_val_ptr, void* heff, double* row_energy,
                     void* stream) {
  g_launches = 0;
  int st = check_drop(drop);
  if (st) return st;
  if (drop->n_systems == 0) return KZ_OK;
  if (!row_val_ptr || !heff || !row_energy) return fail(KZ_ERR_INVALID, "outputs must be non-null");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t rows = (size_t)drop->n_systems * drop->n_users;
  const int wpb = 8;
  const unsigned grid = (unsigned)((rows + wpb - 1) / wpb);
  if (drop->dtype == KZ_C128)
    kz_channel_synth_kernel<double2><<<grid, 32 * wpb, 0, s>>>(*drop, row_val_ptr, (double2*)heff, row_energy);
  else
    kz_channel_synth_kernel<float2><<<grid, 32 * wpb, 0, s>>>(*drop, row_val_ptr, (float2*)heff, row_energy);
  g_launches = 1;
  return cuda_check("kz_channel_synth");
}

int kz_partition_counts(const kz_drop* drop, int32_t* coupled_cnt, int32_t* orth_cnt, int32_t* non_union_size,
                        uint8_t* inset, void* stream) {
  g_launches = 0;
  int st = check_drop(drop);
  if (st) return st;
  if (drop->n_systems == 0) return KZ_OK;
  if (!coupled_cnt || !orth_cnt || !non_union_size || !inset) return fail(KZ_ERR_INVALID, "outputs must be non-null");
  const size_t smem = partition_smem(drop->n_users, drop->n_antennas);
  if (cudaFuncSetAttribute(kz_partition_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return fail(KZ_ERR_UNSUPPORTED, "partition: K=%d too large for shared memory", drop->n_users);
  kz_partition_kernel<<<drop->n_systems, 256, smem, (cudaStream_t)stream>>>(
      *drop, 0, coupled_cnt, orth_cnt, non_union_size, inset, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
  g_launches = 1;
  return cuda_check("kz_partition_counts");
}

int kz_partition_fill(const kz_drop* drop, const int32_t* coupled_ptr, const int32_t* orth_ptr,
                      const int32_t* non_ptr, int32_t* coupled_idx, int32_t* orth_idx, int32_t* non_idx,
                      void* stream) {
  g_launches = 0;
  int st = check_drop(drop);
  if (st) return st;
  if (drop->n_systems == 0) return KZ_OK;
  if (!coupled_ptr || !orth_ptr || !non_ptr || !coupled_idx)
    return fail(KZ_ERR_INVALID, "CSR arrays must be non-null");
  const size_t smem = partition_smem(drop->n_users, drop->n_antennas);
  if (cudaFuncSetAttribute(kz_partition_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return fail(KZ_ERR_UNSUPPORTED, "partition: K=%d too large for shared memory", drop->n_users);
  kz_partition_kernel<<<drop->n_systems, 256, smem, (cudaStream_t)stream>>>(
      *drop, 1, nullptr, nullptr, nullptr, nullptr, coupled_ptr, orth_ptr, non_ptr, coupled_idx, orth_idx, non_idx);
  g_launches = 1;
  return cuda_check("kz_partition_fill");
}

}  // extern "C"

// ------------------------------------------------------------------ per-call step primitives
namespace {

int check_prim(const kz_problem* p, int32_t system, const void* a, const void* b2, const void* c) {
  int st = check_problem(p);
  if (st) return st;
  if (system < 0 || system >= p->n_systems)
    return fail(KZ_ERR_INVALID, "system %d out of range [0, %d)", (int)system, (int)p->n_systems);
  if (!a || !b2 || !c) return fail(KZ_ERR_INVALID, "state arrays must be non-null");
  return KZ_OK;
}

}  // namespace

extern "C" {

int kz_residual_refresh(const kz_problem* prob, int32_t system, int32_t rhs, const void* col, const void* coef,
                        void* resid, const int32_t* rows, int32_t n_rows, int32_t dense, void* stream) {
  g_launches = 0;
  int st = check_prim(prob, system, col, coef, resid);
  if (st) return st;
  if (rhs < 0 || rhs >= prob->n_users) return fail(KZ_ERR_INVALID, "rhs index %d out of range", (int)rhs);
  if (n_rows < 0 || (!rows && n_rows > prob->n_users)) return fail(KZ_ERR_INVALID, "bad row count %d", (int)n_rows);
  if (n_rows == 0) return KZ_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (prob->dtype == KZ_C128)
    kz_prim_refresh<double2><<<1, PRIM_THREADS, 0, s>>>(*prob, system, rhs, (const double2*)col,
                                                         (const double2*)coef, (double2*)resid, rows, n_rows, dense);
  else
    kz_prim_refresh<float2><<<1, PRIM_THREADS, 0, s>>>(*prob, system, rhs, (const float2*)col, (const float2*)coef,
                                                        (float2*)resid, rows, n_rows, dense);
  g_launches = 1;
  return cuda_check("kz_residual_refresh");
}

int kz_project_rows(const kz_problem* prob, int32_t system, void* col, void* coef, void* resid,
                    const int32_t* rows, int32_t n_rows, void* stream) {
  g_launches = 0;
  int st = check_prim(prob, system, col, coef, resid);
  if (st) return st;
  if (n_rows < 0 || (n_rows > 0 && !rows)) return fail(KZ_ERR_INVALID, "rows must be non-null");
  if (n_rows == 0) return KZ_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (prob->dtype == KZ_C128)
    kz_prim_project<double2><<<1, PRIM_THREADS, 0, s>>>(*prob, system, (double2*)col, (double2*)coef,
                                                         (double2*)resid, rows, n_rows);
  else
    kz_prim_project<float2><<<1, PRIM_THREADS, 0, s>>>(*prob, system, (float2*)col, (float2*)coef, (float2*)resid,
                                                        rows, n_rows);
  g_launches = 1;
  return cuda_check("kz_project_rows");
}

int kz_ahk_step(const kz_problem* prob, int32_t system, void* col, void* coef, const void* resid, const void* phi,
                const int32_t* rows, int32_t n_rows, const int32_t* span, int32_t n_span, int32_t* stepped,
                void* stream) {
  g_launches = 0;
  int st = check_prim(prob, system, col, coef, resid);
  if (st) return st;
  if (!phi || !rows || n_rows < 1) return fail(KZ_ERR_INVALID, "ahk_step needs phi and at least one row");
  if (span && n_span < 0) return fail(KZ_ERR_INVALID, "bad span size %d", (int)n_span);
  const size_t smem = (size_t)prob->n_antennas * (prob->dtype == KZ_C128 ? 16 : 8);
  int dev = 0, maxsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (smem + 1024 > (size_t)maxsm)
    return fail(KZ_ERR_UNSUPPORTED, "ahk_step: %d antennas exceed the shared-memory aggregation buffer",
                (int)prob->n_antennas);
  cudaStream_t s = (cudaStream_t)stream;
  if (prob->dtype == KZ_C128) {
    cudaFuncSetAttribute(kz_prim_ahk<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kz_prim_ahk<double2><<<1, PRIM_THREADS, smem, s>>>(*prob, system, (double2*)col, (double2*)coef,
                                                        (const double2*)resid, (const double2*)phi, rows, n_rows,
                                                        span, n_span, stepped);
  } else {
    cudaFuncSetAttribute(kz_prim_ahk<float2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kz_prim_ahk<float2><<<1, PRIM_THREADS, smem, s>>>(*prob, system, (float2*)col, (float2*)coef,
                                                       (const float2*)resid, (const float2*)phi, rows, n_rows, span,
                                                       n_span, stepped);
  }
  g_launches = 1;
  return cuda_check("kz_ahk_step");
}

}  // extern "C"

