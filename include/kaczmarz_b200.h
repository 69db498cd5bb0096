/*
 * kaczmarz_b200.h — C ABI of the B200-native batched Kaczmarz precoding path.
 *
 * The reference (arXiv 2501.10689, `kaczprec`) is pure Python and has no FFI
 * layer; its boundary is the Python API of `kaczprec.solvers` / `rzf` /
 * `assembly` / `metrics`.  Each entry point below replaces one group of those
 * calls for a whole batch of independent systems (realizations/subcarriers):
 *
 *   kz_solve     <- run_precoding   (pkg/src/kaczprec/solvers.py:556-623)
 *                   solve / solve_all (solvers.py:460-537)
 *                   InstanceRun.step + step primitives (solvers.py:143-423)
 *   kz_rzf       <- rzf_precoder / auxiliary_matrix (pkg/src/kaczprec/rzf.py:38-83)
 *   kz_residual_refresh / kz_project_rows / kz_ahk_step
 *                <- residual_refresh, rk_step + orthogonal_block_step, ahk_step (solvers.py:143-309, 312-332):
 *                   the per-call step primitives on one rhs of one system (InstanceRun.step's building blocks)
 *   kz_epilogue  <- assemble_dense / assemble_vr (pkg/src/kaczprec/assembly.py:51-92),
 *                   nmse / spectral_efficiency (pkg/src/kaczprec/metrics.py:44-78)
 *
 * Conventions
 *  - Plain C types only; every device buffer is caller-owned (the library
 *    never allocates device memory) and passed as a raw device pointer.
 *  - Complex arrays are interleaved (re, im); element type is double for
 *    KZ_C128 and float for KZ_C64.
 *  - All calls are asynchronous on `stream` (a cudaStream_t passed as void*;
 *    NULL = legacy default stream).  They return KZ_OK or a negative status;
 *    kz_last_error() gives a thread-local message.  No exceptions cross the ABI.
 *  - Non-convergence is a flag in the outputs, never an error (solvers.py:477,498-505).
 */
#ifndef KACZMARZ_B200_H
#define KACZMARZ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KZ_ABI_VERSION 8

/* status codes */
#define KZ_OK 0
#define KZ_ERR_INVALID (-1)   /* bad argument; reference raises ValueError */
#define KZ_ERR_CUDA (-2)      /* CUDA runtime error */
#define KZ_ERR_NOT_PD (-3)    /* Gram not positive definite; reference raises LinAlgError (rzf.py:55-59) */
#define KZ_ERR_WORKSPACE (-4) /* workspace too small */
#define KZ_ERR_UNSUPPORTED (-5)

/* schemes, in the order of SCHEMES (solvers.py:39), then the extension the BASELINE cfg3 asks for */
enum kz_scheme { KZ_URK = 0, KZ_SWOR_ERK = 1, KZ_GK = 2, KZ_GRK = 3, KZ_VR_OGRK = 4, KZ_AHK = 5, KZ_VR_OAHK = 6,
                 /* grouped VR-OAHK (no reference counterpart; CPU restatement oracle/grouped.py): per iteration an
                    exact block step on each orthogonal group O_1..O_g, then the non-orthogonal rows aggregated in
                    consecutive blocks of at most kz_problem.agg_cap rows.  g = 1 and agg_cap >= |N| is vr-oahk. */
                 KZ_VR_OAHK_G = 7 };
enum kz_dtype { KZ_C128 = 0, KZ_C64 = 1 };

/* stopping drivers */
enum kz_stop_mode {
  KZ_STOP_LOCKSTEP = 0, /* run_precoding: all K rhs advance per outer iteration; stop when
                           NMSE(M/||M||, F_ref) < epsilon (epsilon = 0: fixed T) (solvers.py:587-603) */
  KZ_STOP_RESIDUAL = 1, /* solve/solve_all mode="residual": ||r_true||_2 <= epsilon (solvers.py:494-497) */
  KZ_STOP_ORACLE = 2    /* solve/solve_all mode="oracle": ||q - v_ref||/||v_ref|| < epsilon (solvers.py:488-493) */
};

/* where the random row draws come from */
enum kz_rng_kind {
  KZ_RNG_NONE = 0,           /* deterministic schemes (gk, ahk, vr-oahk) */
  KZ_RNG_HOST_UNIFORM = 1,   /* u[b][rhs][s] fp64: one Generator.random() per greedy-weighted pick */
  KZ_RNG_HOST_INDEX = 2,     /* idx[b][rhs][s] int32: host-evaluated uniform / energy-swor picks */
  KZ_RNG_PHILOX = 3          /* on-device Philox4x32-10 keyed by (seed, system_base + b, rhs, draw) */
};

/*
 * One batch of B independent systems sharing (K, Nt).  Row i of system b has
 * support Gamma_bi given as a list of contiguous antenna segments and its
 * restricted channel h_bi = H_b[Gamma_bi, i] packed contiguously
 * (AugmentedSystem.supports / eff_rows, solvers.py:80-89).
 */
typedef struct kz_problem {
  int32_t n_systems;   /* B */
  int32_t n_users;     /* K (rows and right-hand sides) */
  int32_t n_antennas;  /* Nt */
  int32_t dtype;       /* kz_dtype of heff and of every complex output */
  /* supports: row r = b*K + i owns segments [row_seg_ptr[r], row_seg_ptr[r+1]) */
  const int32_t* row_seg_ptr;   /* [B*K+1] */
  const int32_t* seg_start;     /* [n_seg] first antenna of the segment */
  const int32_t* seg_len;       /* [n_seg] */
  const int64_t* row_val_ptr;   /* [B*K+1] offset of h_bi in heff (complex elements) */
  const void* heff;             /* packed complex values */
  const double* row_energy;     /* [B*K] e_bi = ||h_bi||^2 + reg_b (solvers.py:90) */
  const double* reg;            /* [B] ridge weight xi_b */
  /* VR partition (vrgraph.py:84-114), only read by vr-ogrk / vr-oahk */
  const int32_t* coupled_ptr;   /* [B*K+1] into coupled_idx; X_bi ascending */
  const int32_t* coupled_idx;
  const int32_t* orth_ptr;      /* [B+1] into orth_idx; O_b ascending */
  const int32_t* orth_idx;
  const int32_t* non_ptr;       /* [B+1] into non_idx; N_b ascending */
  const int32_t* non_idx;
  const int32_t* non_union_size;/* [B] |union of N_b supports| (flop charge of ahk_step) */
  /* shape hints, set by the packer (trusted): enable the register-resident fast path */
  int32_t max_support;          /* max_r |Gamma_r| */
  int32_t flags;                /* KZ_PROBLEM_CONTIGUOUS: every row is exactly one segment */
  /* max over systems and CTAs of the (row, 32-antenna chunk) pairs one CTA of the large-array cluster path
     holds, for 128- / 256-antenna CTAs in its block-interleaved layout (CL = ceil(Nt / width) CTAs; with
     CL > 1 CTA c owns two blocks of width/2 antennas, block j starting at antenna (j*CL + c) * width/2);
     contiguous supports only, 0 = unknown (cluster path disabled) */
  int32_t slice_pairs_128;
  int32_t slice_pairs_256;
  /* max over systems and CTAs of the rows with at least one piece in one CTA of the same layouts (0 = use
     min(K, pairs)) */
  int32_t slice_rows_128;
  int32_t slice_rows_256;
  /* KZ_VR_OAHK_G only: the orthogonal rows of system b (orth_idx[orth_ptr[b] .. orth_ptr[b+1])) form the groups
     [ogrp_ptr[j], ogrp_ptr[j+1]) for j in [ogrp_sys[b], ogrp_sys[b+1]) (absolute offsets into orth_idx, each group
     ascending and pairwise VR-disjoint); the non-orthogonal rows are aggregated in consecutive blocks of at most
     agg_cap rows */
  const int32_t* ogrp_sys;      /* [B+1] */
  const int32_t* ogrp_ptr;      /* [total groups + 1] */
  int32_t agg_cap;
  int32_t _pad0;
  /* element range [val_lo, val_hi) of heff the batch's rows occupy (= row_val_ptr[0], row_val_ptr[B*K] for dense
     packing).  When known (val_hi > val_lo) the complex64 on-chip kernels stage H_eff into shared memory with TMA
     tensor copies over that range; 0, 0 = unknown (asynchronous-copy staging) */
  int64_t val_lo;
  int64_t val_hi;
} kz_problem;

#define KZ_PROBLEM_CONTIGUOUS 1
/* kz_epilogue only: the workspace already holds G0 = H^H H of this problem from an earlier kz_epilogue call
   on the same workspace (the Gram-form path; H is the same, so several V of one batch share it) */
#define KZ_PROBLEM_GRAM_CACHED 2

typedef struct kz_stop {
  int32_t mode;         /* kz_stop_mode */
  int32_t max_iters;    /* cap: outer iterations (LOCKSTEP) or per-rhs iterations (RESIDUAL/ORACLE) */
  int32_t check_every;  /* StoppingRule.check_every (>= 1) */
  int32_t _pad;
  double epsilon;       /* LOCKSTEP: NMSE threshold (0 = fixed T); else StoppingRule.epsilon (> 0) */
  const double* f_ref;  /* LOCKSTEP with epsilon > 0 or traces: [B][Nt][K] complex128 F_ref */
  const double* v_ref;  /* ORACLE: [B][K][K] complex128, column c = reference for rhs c */
  const uint8_t* rhs_mask; /* optional [B*K]; 0 = leave that rhs untouched (solve() on one column) */
} kz_stop;

typedef struct kz_rng {
  int32_t kind;          /* kz_rng_kind */
  int32_t stream_len;    /* draws per (b, rhs) available in this call (HOST_*) */
  int64_t stream_base;   /* global draw index of element 0 (chunked resumption) */
  const double* uniforms;/* HOST_UNIFORM: [B][K][stream_len] */
  const int32_t* indices;/* HOST_INDEX:   [B][K][stream_len] */
  uint64_t seed;         /* PHILOX key */
  int64_t system_base;   /* PHILOX: global index of system 0 of this batch.  The draws of a system are keyed by
                            its global index, so a realization's row stream does not depend on how the
                            realizations are chunked or sharded across ranks (the reference's worker-count
                            invariance, pkg/README.md:68-70, tests/test_experiments.py:139-146) */
} kz_rng;

typedef struct kz_out {
  void* v;                  /* [B][K][K] complex (dtype): v[b][i][c] = coef_i of rhs c (PrecodingRun.v) */
  int32_t* iters;           /* [B*K] SolverState.iters per rhs */
  uint8_t* converged;       /* [B*K] per-rhs convergence (solve) */
  uint8_t* done;            /* [B*K] greedy/no-op termination flag (InstanceRun.done) */
  int32_t* noop_steps;      /* [B*K] */
  int64_t* flops;           /* [B*K] FlopCounter.total per rhs (metrics.py:25-41) */
  int32_t* n_outer;         /* [B] LOCKSTEP outer iterations t (PrecodingRun.n_iters) */
  uint8_t* sys_converged;   /* [B] LOCKSTEP convergence */
  uint8_t* paused;          /* [B*K] optional: rhs ran out of host draws (resume with next chunk) */
  int32_t* rows;            /* optional [B][K][rows_cap]: projected row per RK step */
  int32_t rows_cap;
  int32_t trace_cap;        /* length of the optional traces below */
  /* LOCKSTEP: [B][trace_cap], one entry per outer iteration (PrecodingRun traces):
       nmse of M/||M|| vs F_ref, ||I - H^H M - xi Q||_F, sum of per-rhs flop counters.
     RESIDUAL/ORACLE: [B*K][trace_cap], one entry per check (RunTrace of solve):
       ||q - v_ref||/||v_ref|| (oracle mode), fresh ||r||_2, the rhs's flop counter. */
  double* nmse_trace;
  double* resid_trace;
  int64_t* flops_trace;
  int32_t* n_checks;        /* optional [B*K] (RESIDUAL/ORACLE): entries written per rhs */
  void* iterates;           /* optional [B][K rhs][Nt] complex (dtype): final iterate m (SolverState.col) */
} kz_out;

/* Bytes of device workspace that is enough for any kz_solve call on this problem (the global-memory kernel's
   iterates M, residuals and per-rhs scratch; the workspace doubles as its resumable solver state). */
size_t kz_solve_workspace_bytes(const kz_problem* prob, const kz_stop* stop);

/* Bytes the kz_solve(prob, scheme, stop, rng, out, resume = 0) call would need for the kernel it dispatches to:
   the on-chip kernels (contiguous supports, fixed T or per-rhs residual tolerance) keep every iterate in
   registers / shared memory / TMEM and need only B*K int32 of stop bookkeeping, so a batch as large as
   BASELINE cfg4 (B = 16384, K = 256, Nt = 4096) runs in one call; the cluster kernel's streamed variant (residual-
   mode aggregation schemes) adds a chunk-padded copy of H_eff (B*K*ceil(max_support/32 + 1)*32 complex64; with a
   smaller workspace the staged variant runs instead); the global-memory kernel needs kz_solve_workspace_bytes.
   Decides without launching (device attributes of the current device). */
size_t kz_solve_workspace_bytes_for(const kz_problem* prob, int32_t scheme, const kz_stop* stop, const kz_rng* rng,
                                    const kz_out* out);

/* Byte offset in that workspace of the stored row residuals (SolverState.resid, solvers.py:112-136) after a
   complex128 KZ_STOP_RESIDUAL / KZ_STOP_ORACLE solve: [B*K rhs][K] complex of prob->dtype, rhs-major. */
size_t kz_solve_resid_offset(const kz_problem* prob);

/* Run scheme over every (system, rhs).  resume = 0 initialises the state
   (SolverState.initial, solvers.py:129-136); resume = 1 continues from the
   workspace (next host-stream chunk). */
int kz_solve(const kz_problem* prob, int32_t scheme, const kz_stop* stop, const kz_rng* rng,
             kz_out* out, void* workspace, size_t workspace_bytes, int32_t resume, void* stream);

/* Batched direct RZF (rzf.py:38-83): Gram H^H H + reg I from the packed rows,
   Cholesky, V = Gram^{-1}, F = beta H V with ||F||_F = 1.  Always complex128.
   v_out [B][K][K], f_out [B][Nt][K] (may be NULL), beta_out [B].
   Returns KZ_ERR_NOT_PD if any Gram is not positive definite (status per
   system in pd_ok [B], may be NULL). */
size_t kz_rzf_workspace_bytes(const kz_problem* prob);
int kz_rzf(const kz_problem* prob, double* v_out, double* f_out, double* beta_out,
           uint8_t* pd_ok, void* workspace, size_t workspace_bytes, void* stream);

/* Precoder epilogue for a batch of auxiliary solutions V (assembly.py:51-92,
   metrics.py:44-78):
     beta = 1/||H V||_F, F = beta H V (blocked over the rows covering each antenna,
     identical to the dense product because H is zero off-support);
     nmse = ||F_ref - F||_F / ||F_ref||_F with F_ref = beta_ref H V_ref (never materialised);
     rates_k = log2(1 + |h_k^H f_k|^2 / (sum_{i!=k} |h_k^H f_i|^2 + 1/snr_linear)), via
     H^H F = beta (H^H H) V.
   v [B][K][K] (prob->dtype); f_out [B][Nt][K] (prob->dtype, NULL = not stored);
   v_ref [B][K][K] complex128 + beta_ref [B] (NULL = no NMSE); snr_linear [B]
   (NULL = no rates); beta_out [B], nmse_out [B], rates_out [B][K], sum_rate_out [B]
   each may be NULL. */
size_t kz_epilogue_workspace_bytes(const kz_problem* prob);
/* 1 if kz_epilogue on this problem takes the Gram form (contiguous VRs, K >= 32, F not stored: every output is a
   quadratic form in G0 = H^H H, which the workspace then holds and KZ_PROBLEM_GRAM_CACHED may reuse), else 0 */
int32_t kz_epilogue_uses_gram(const kz_problem* prob, int32_t want_f);
int kz_epilogue(const kz_problem* prob, const void* v, void* f_out, const double* v_ref, const double* beta_ref,
                const double* snr_linear, double* beta_out, double* nmse_out, double* rates_out,
                double* sum_rate_out, void* workspace, size_t workspace_bytes, void* stream);

/*
 * On-device input preparation for contiguous-VR near-field drops: a batch of B
 * systems described by their user drop; the packed layout of kz_problem is built on the device.
 */
typedef struct kz_drop {
  int32_t n_systems;          /* B */
  int32_t n_users;            /* K */
  int32_t n_antennas;         /* Nt (ULA, element n at x_n = (n - (Nt-1)/2) * element_spacing) */
  int32_t dtype;              /* kz_dtype of heff */
  double element_spacing;     /* metres (lambda_carrier / 2 in the BASELINE configs) */
  const double* wavelength;   /* [B] wavelength of each system (per subcarrier for wideband OFDM) */
  const double* r0;           /* [B*K] user distance to the array centre (m) */
  const double* theta;        /* [B*K] user angle from broadside (rad) */
  const int32_t* vr_start;    /* [B*K] first visible antenna */
  const int32_t* vr_len;      /* [B*K] visible antennas (>= 1) */
  const double* reg;          /* [B] ridge weight xi */
} kz_drop;

/* heff rows lambda/(4 pi r_n) exp(-j 2 pi r_n / lambda) on [vr_start, vr_start + vr_len), unit-norm per user,
   at heff + row_val_ptr[b*K+i] (caller-computed exclusive prefix of vr_len, [B*K+1]); row_energy [B*K] =
   ||h_bi||^2 + reg_b.  Replaces host channel generation + packing (channel.py, solvers.py:80-92). */
int kz_channel_synth(const kz_drop* drop, const int64_t* row_val_ptr, void* heff, double* row_energy, void* stream);

/* VR partition on the device (vrgraph.py:31-114).  Pass 1 counts: coupled_cnt [B*K] = |X_bi|,
   orth_cnt [B] = |O_b|, non_union_size [B], inset [B*K] (1 = O, 2 = N).  The caller forms the exclusive
   prefixes coupled_ptr [B*K+1], orth_ptr [B+1], non_ptr [B+1] (N_b has K - |O_b| rows); pass 2 fills
   coupled_idx, orth_idx, non_idx in ascending order. */
int kz_partition_counts(const kz_drop* drop, int32_t* coupled_cnt, int32_t* orth_cnt, int32_t* non_union_size,
                        uint8_t* inset, void* stream);
int kz_partition_fill(const kz_drop* drop, const int32_t* coupled_ptr, const int32_t* orth_ptr,
                      const int32_t* non_ptr, int32_t* coupled_idx, int32_t* orth_idx, int32_t* non_idx,
                      void* stream);

/*
 * Per-call step primitives on ONE right-hand side of system `system` of `prob` (solvers.py:143-332).  The
 * state is SolverState (solvers.py:112-136) in device memory, prob->dtype complex: col [Nt], coef [K],
 * resid [K]; rows / span are device int32 index arrays.  Flop charges and iteration / no-op counters are the
 * caller's (they depend only on sizes, metrics.py:25-41).
 */
/* residual_refresh(state, sys, rows, use_vr) (solvers.py:143-170): resid_i = s_i - h_i^H col - reg coef_i for
   the n_rows rows (rows = NULL: i = 0..n_rows-1); dense = 1 evaluates the h_adj @ col form (:149-153). */
int kz_residual_refresh(const kz_problem* prob, int32_t system, int32_t rhs, const void* col, const void* coef,
                        void* resid, const int32_t* rows, int32_t n_rows, int32_t dense, void* stream);
/* rk_step (solvers.py:173-188) for n_rows = 1, orthogonal_block_step (:312-332) for a row list: per row, in
   order, gamma = resid_i / e_i, col[Gamma_i] += gamma h_i, coef_i += gamma, resid_i = 0. */
int kz_project_rows(const kz_problem* prob, int32_t system, void* col, void* coef, void* resid,
                    const int32_t* rows, int32_t n_rows, void* stream);
/* ahk_step (solvers.py:257-309) with weights phi [K] (complex, prob->dtype) on the sorted rows: y = sum phi_i h_i,
   den = ||y||^2 + reg ||phi_rows||^2; den == 0 leaves the state untouched and writes *stepped = 0 (device
   int32); else gamma = phi_rows^H resid_rows / den, col[span] += gamma y[span] (span = the support union, or
   NULL for every antenna), coef[rows] += gamma phi_rows, *stepped = 1.  The caller handles the empty / all-zero
   phi no-op (:270-273) before calling. */
int kz_ahk_step(const kz_problem* prob, int32_t system, void* col, void* coef, const void* resid, const void* phi,
                const int32_t* rows, int32_t n_rows, const int32_t* span, int32_t n_span, int32_t* stepped,
                void* stream);

/* Number of kernels the last kz_* call on this thread launched (benchmark
   bookkeeping for the gpu_launches count). */
int32_t kz_last_launch_count(void);
/* 1 if the last kz_solve on this thread staged H_eff into shared memory with TMA tensor copies (complex64
   on-chip kernels with kz_problem.val_lo/val_hi set), else 0 (evidence for the staging path) */
int32_t kz_last_tma_staging(void);

const char* kz_last_error(void);
int32_t kz_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* KACZMARZ_B200_H */
