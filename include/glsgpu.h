/*
 * glsgpu.h -- the C-ABI drop-in boundary of the B200-native GLS-PCG (PCG-Aug, SUR) solver.
 *
 * Plain pointers and sizes only (no torch / CUDA types in the signatures).  Every entry point
 * replaces one piece of the reference's C++ hot path (citations are /root/reference paths):
 *
 *   glsgpu_sur_create / _create_device   make_sur + sur_preconditioner (per-block Householder QR)
 *                                        proj/include/gls/structured.hpp:63,105-108;
 *                                        proj/src/structured.cpp:97-105,416-453,479-486
 *   glsgpu_apply_pi / _xstar_t / _xstar  IndefinitePreconditioner::apply_pi/apply_xstar_t/apply_xstar
 *                                        proj/include/gls/preconditioner.hpp:36-38;
 *                                        proj/src/preconditioner.cpp:9-28, structured.cpp:307-340
 *   glsgpu_sigma_apply                   SymmetricOperator::apply, Kronecker branch
 *                                        proj/include/gls/operators.hpp:18,22; proj/src/operators.cpp:42-50
 *   glsgpu_operator_norm_probe           operator_norm_probe  proj/include/gls/pcg.hpp:132; pcg.cpp:233-244
 *   glsgpu_sur_solve                     pcg_aug(embed_sur(sur), *sur_preconditioner(sur), w1, z1, cfg,
 *                                        true_beta)  proj/include/gls/pcg.hpp:80-83; proj/src/pcg.cpp:36-229,346-350
 *   glsgpu_counters / _reset_counters    IndefinitePreconditioner::counters / reset_apply_counters
 *                                        proj/include/gls/preconditioner.hpp:40-41; preconditioner.cpp:30-35
 *   glsgpu_mvrglm_create                 make_mvrglm + mvrglm_preconditioner (+ embed_mvrglm's operator layout)
 *                                        proj/include/gls/structured.hpp:33-50,96-100;
 *                                        proj/src/structured.cpp:63-95,365-414,468-477
 *   glsgpu_mv_reduce                     mv_reduce  proj/include/gls/structured.hpp:76; structured.cpp:121-130
 *   glsgpu_sur_reduce                    sur_reduce proj/include/gls/structured.hpp:80-81; structured.cpp:132-178
 *   glsgpu_pcg_ne                        pcg_normal_equations(embed_sur(sur), nullptr, cfg, true_beta)
 *                                        proj/include/gls/pcg.hpp; proj/src/pcg.cpp:364-511
 *
 * Errors: every call returns a status code; the codes map 1:1 onto the reference's gls::Error
 * subclasses (proj/include/gls/errors.hpp:10-88) and glsgpu_last_error_message() holds the text.
 * There is no CPU fallback: without a CUDA device, creation fails with GLSGPU_ERR_NO_DEVICE.
 *
 * Layouts (as the reference, proj/include/gls/dense_matrix.hpp:13-15): column-major.  X is the
 * concatenation [X_0 | ... | X_{G-1}] as one M x n matrix (n = sum n_i); Y is M x G; Omega is G x G;
 * every m-vector (m = G*M) is stacked equation-major, i.e. equation b owns [b*M, (b+1)*M).
 */
#ifndef GLSGPU_H
#define GLSGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (gls::Error subclasses, proj/include/gls/errors.hpp). */
enum {
  GLSGPU_OK = 0,
  GLSGPU_ERR_DIMENSION_MISMATCH = 1,  /* gls::DimensionMismatch */
  GLSGPU_ERR_RANK_DEFICIENT = 2,      /* gls::RankDeficient ("block i is rank deficient") */
  GLSGPU_ERR_SINGULAR_D = 3,          /* gls::SingularD (non-positive block scale) */
  GLSGPU_ERR_SINGULAR_TRIANGULAR = 4, /* gls::SingularTriangular */
  GLSGPU_ERR_SINGULAR_COVARIANCE = 5, /* gls::SingularCovariance (PCG-NE: Sigma not positive definite) */
  GLSGPU_ERR_CUDA = 10,               /* CUDA runtime failure */
  GLSGPU_ERR_NO_DEVICE = 11,          /* no CUDA device: there is no CPU fallback */
  GLSGPU_ERR_OUT_OF_MEMORY = 12,
  GLSGPU_ERR_UNSUPPORTED = 13,        /* shape outside this build's kernels (e.g. n_i > 512, G > 512) */
  GLSGPU_ERR_INVALID = 14,            /* null handle / bad argument */
  GLSGPU_ERR_NCCL = 15
};

/* gls::Termination (proj/include/gls/glm.hpp:26), same order. */
enum { GLSGPU_CONVERGED = 0, GLSGPU_BREAKDOWN = 1, GLSGPU_STAGNATION = 2, GLSGPU_MAXITER = 3, GLSGPU_DIRECT = 4 };

/* How X*v enters the residual update r -= lambda (Sigma u + X v)  (proj/src/pcg.cpp:154-155). */
enum {
  GLSGPU_XV_X = 0,  /* reference-faithful: the original X times v (bitwise the reference's row sums) */
  GLSGPU_XV_QR = 1  /* Q (R v) with R v kept by the recurrence s = Q'r + mu s: X is not streamed */
};

/* gls::PcgConfig (proj/include/gls/pcg.hpp:12-30) plus device-execution knobs. */
typedef struct {
  double tol_rel;            /* stop when c_{i+1} <= tol_rel^2 c_1 */
  int64_t max_iter;          /* 0 -> m - n + 1 */
  double breakdown_tol;      /* 1e-14 */
  int64_t stagnation_window; /* 5 */
  double growth_tol;         /* 1e4 */
  int64_t growth_window;     /* 10 */
  int64_t record_z_every;    /* 1 */
  /* --- device knobs (not in the reference) --- */
  int32_t diag_every;        /* trace diagnostics (aug_residual_norm, dual_feas_norm, rmse) every k rows;
                                1 = every row as the reference; 0 = row 0 and the terminating row only */
  int32_t xv_mode;           /* GLSGPU_XV_X or GLSGPU_XV_QR */
  int32_t graph_chunk;       /* PCG iterations per CUDA-graph launch (0 = auto) */
  int32_t kernel_timing;     /* 1 = record CUDA events around every streaming pass (glsgpu_kernel_stats) */
  int32_t kron_fma;          /* Kronecker pass of the FP64-bound shapes (128 < G <= 256): 0 = separate
                                multiply and add, bitwise the reference's operator* (default); 1 = one
                                fused multiply-add per term (half the FP64 instructions; one rounding per
                                term instead of two) */
  int32_t sw_mode;           /* 0 = Sigma w by the reference's recurrence sw -= lambda su (pcg.cpp:152); 1 = Sigma w
                                formed where it is read (diagnostics rows, the exit's b = X*'(y - Sigma w_sel)):
                                pass A then moves 3 fewer M x G vectors.  Takes effect with kron_fma on the
                                DMMA pass A (128 < G <= 256) and diag_every <= 0 */
  int32_t fused_c;           /* 1 = Sigma pr formed on the tensor cores inside pass C (one sweep with Pi r) and
                                Sigma u = Sigma pr + mu Sigma u carried by recurrence, so pass A is element-wise.
                                Takes effect with sw_mode 1 and tile-contiguous Q (n_i <= 32) */
} glsgpu_pcg_config;

/* gls::PcgTraceRow (proj/include/gls/pcg.hpp:32-39).  Diagnostics not computed are NaN. */
typedef struct {
  int64_t iter;
  double c;
  double aug_residual_norm;
  double dual_feas_norm;
  double rmse;
  int64_t elapsed_ns;
} glsgpu_trace_row;

/* GlsSolution / PcgTrace scalars (proj/include/gls/glm.hpp:30-37, pcg.hpp:41-51). */
typedef struct {
  int64_t iterations;
  int32_t termination;
  int32_t w1_projected;
  int64_t breakdown_iteration; /* -1 when absent */
  double residual_seminorm;
  int64_t n_rows;              /* trace rows (iterations + 1) */
  double sigma_scale;          /* operator_norm_probe(Sigma) used by the breakdown test */
  double solve_ms;             /* device time of the solve (CUDA events on the solver stream) */
} glsgpu_result;

/* gls::CostCounters (proj/include/gls/preconditioner.hpp:15-22). */
typedef struct {
  uint64_t factorizations;
  uint64_t factor_multiplies;
  uint64_t pi_applies;
  uint64_t xstar_t_applies;
  uint64_t xstar_applies;
  uint64_t apply_multiplies;
} glsgpu_counters_t;

/* Per streaming pass timing (kernel_timing = 1). */
typedef struct {
  char name[32];
  int64_t launches;
  double total_ms;
  double bytes_per_launch;     /* algorithmic bytes of one launch */
} glsgpu_kernel_stat;

typedef struct glsgpu_sur glsgpu_sur; /* opaque: one SUR operator resident on one device */

int glsgpu_device_count(int* count);
const char* glsgpu_last_error_message(void);
const char* glsgpu_version(void);

/* make_sur + sur_preconditioner from HOST buffers (copied to the device; the QR runs there).
 * block_scale may be NULL (D = I).  On RankDeficient / SingularD, *bad_block gets the block. */
int glsgpu_sur_create(int G, int64_t M, const int64_t* n_i, const double* X, const double* Y,
                      const double* omega, const double* block_scale, int device, glsgpu_sur** out,
                      int* bad_block);

/* Same from DEVICE-resident X (ld >= M, column-major) and Y (ld >= M): no host copy of the big
 * inputs.  The caller keeps X_dev / Y_dev alive for the handle's lifetime. */
int glsgpu_sur_create_device(int G, int64_t M, const int64_t* n_i, const double* X_dev, int64_t ldx,
                             const double* Y_dev, int64_t ldy, const double* omega, const double* block_scale,
                             int device, glsgpu_sur** out, int* bad_block);

/* New X (M x n) and Y (M x G) from HOST buffers for a handle made by glsgpu_sur_create or
 * glsgpu_sur_create_sharded_host (same shapes; a sharded handle takes this rank's rows): upload and refactor,
 * reusing the handle's device memory and factorisation plan (create once, solve many).  This is make_sur +
 * sur_preconditioner for the next model (proj/src/structured.cpp:97-105,416-453) without reallocating. */
int glsgpu_sur_update(glsgpu_sur* h, const double* X, const double* Y, int* bad_block);

/* Pipelined form of glsgpu_sur_update for a stream of models: glsgpu_sur_stage queues the NEXT model's X and Y
 * (pinned host memory, same shapes) for upload on the handle's copy stream as soon as the current factorisation
 * has consumed the resident X -- so the upload overlaps the current solve -- and glsgpu_sur_update_staged makes it
 * current (waits for the copy, refactors).  Between the two, the resident X belongs to the next model: solves
 * must run in xv_mode QR without w1 / z1 (they never read X; the trace diagnostics use Q and R), and
 * glsgpu_sur_refactor / glsgpu_pcg_ne refuse with GLSGPU_ERR_UNSUPPORTED.  X / Y stay untouched by the caller
 * until glsgpu_sur_update_staged returns. */
int glsgpu_sur_stage(glsgpu_sur* h, const double* X, const double* Y);
int glsgpu_sur_update_staged(glsgpu_sur* h, int* bad_block);

/* Re-run the setup QR from the resident X (the per-solve setup cost; bench steps time it). */
int glsgpu_sur_refactor(glsgpu_sur* h, int* bad_block);

int glsgpu_sur_destroy(glsgpu_sur* h);
int glsgpu_sur_dims(const glsgpu_sur* h, int* G, int64_t* M, int64_t* n);
/* The solver's CUDA stream (cudaStream_t as void*), for callers that time on it. */
void* glsgpu_sur_stream(const glsgpu_sur* h);

/* Probe-level operator applies on HOST vectors (sizes m -> m, m -> n, n -> m). */
int glsgpu_apply_pi(glsgpu_sur* h, const double* xi, double* out);
int glsgpu_apply_xstar_t(glsgpu_sur* h, const double* xi, double* out);
int glsgpu_apply_xstar(glsgpu_sur* h, const double* v, double* out);
int glsgpu_sigma_apply(glsgpu_sur* h, const double* x, double* out);
int glsgpu_operator_norm_probe(glsgpu_sur* h, int64_t iters, double* norm);

int glsgpu_counters(const glsgpu_sur* h, glsgpu_counters_t* out);
int glsgpu_reset_apply_counters(glsgpu_sur* h);

/* pcg_aug on the SUR model.  w1 (m), z1 (n), beta_true (n) may be NULL (zeros / no rmse).
 * b_out (n) required; w_out (m) and rows (rows_cap) optional. */
int glsgpu_sur_solve(glsgpu_sur* h, const glsgpu_pcg_config* cfg, const double* w1, const double* z1,
                     const double* beta_true, double* b_out, double* w_out, glsgpu_trace_row* rows,
                     int64_t rows_cap, glsgpu_result* res);

void glsgpu_default_config(glsgpu_pcg_config* cfg);

/* Kernel statistics of the last solve with kernel_timing = 1; returns the number written. */
int glsgpu_kernel_stats(const glsgpu_sur* h, glsgpu_kernel_stat* out, int cap);

/* Kernels this handle has launched so far (CUDA-graph kernel nodes counted per graph launch). */
int glsgpu_launch_count(const glsgpu_sur* h, int64_t* count);

/* Row sharding over several GPUs (one process per GPU) ------------------------
 * Rank r owns rows [row0_r, row0_r + M_local) of every block (any contiguous split; each rank needs
 * at least max n_i rows); Omega, R and every n-vector are replicated.  Per PCG iteration the ranks
 * all-gather three small partial-sum vectors over NCCL (d, u.u | Q'r per block | c, r.r, pr.pr) and
 * reduce them in rank order, so every rank takes bitwise the same decisions.  The setup factorisation works across
 * ranks too: CholeskyQR2 all-gathers the per-rank Gram matrices, its TSQR fallback the per-rank R factors.  Host
 * vectors passed to the probe applies / solve of a sharded handle are the rank's local rows; b is replicated. */
int glsgpu_nccl_unique_id(void* id_out /* 128 bytes (ncclUniqueId) */);
int glsgpu_sur_create_sharded(int G, int64_t M_local, int64_t M_global, const int64_t* n_i, const double* X_dev,
                              int64_t ldx, const double* Y_dev, int64_t ldy, const double* omega,
                              const double* block_scale, int device, const void* nccl_id, int rank, int nranks,
                              glsgpu_sur** out, int* bad_block);
int glsgpu_sur_shard(const glsgpu_sur* h, int* rank, int* nranks, int64_t* M_global);

/* Sharded handle from this rank's HOST rows (X: M_local x n, Y: M_local x G, ld M_local); the handle owns its
 * device copies, so glsgpu_sur_update / _stage / _update_staged serve it (the per-step e2e path at N > 1). */
int glsgpu_sur_create_sharded_host(int G, int64_t M_local, int64_t M_global, const int64_t* n_i, const double* X,
                                   const double* Y, const double* omega, const double* block_scale, int device,
                                   const void* nccl_id, int rank, int nranks, glsgpu_sur** out, int* bad_block);

/* TEST-ONLY in-process rank group: nranks row-shard handles of ONE process on ONE device, each driven by its own
 * host thread, exchange their all-gathers by device-to-device copies ordered with CUDA events and host barriers
 * instead of NCCL (no kernel ever waits on another rank).  It runs the library's real sharded decomposition --
 * cross-rank TSQR level, rank-order sums -- where only one GPU is available; solves run without CUDA graphs.
 * Not a product backend: multi-GPU runs use glsgpu_sur_create_sharded[_host] over NCCL. */
typedef struct glsgpu_local_group glsgpu_local_group;
int glsgpu_local_group_create(int nranks, int device, glsgpu_local_group** out);
int glsgpu_local_group_destroy(glsgpu_local_group* g);
int glsgpu_sur_create_sharded_local(int G, int64_t M_local, int64_t M_global, const int64_t* n_i, const double* X_dev,
                                    int64_t ldx, const double* Y_dev, int64_t ldy, const double* omega,
                                    const double* block_scale, glsgpu_local_group* group, int rank, glsgpu_sur** out,
                                    int* bad_block);

/* Multivariate model with exclusion restrictions (gls::MvRglm) ------------------------------------
 * Y = Z0 B + U, restriction list i = the zero-forced rows of B[:, i] as CSR: equation i restricts parameters
 * ridx[roff[i] .. roff[i + 1]) (strictly increasing, < N0; roff[0] = 0).  The handle is the operator of
 * pcg_aug(embed_mvrglm(mv), *mvrglm_preconditioner(mv[, z_scale, c_scale]), ...): every entry point above
 * (applies, sigma_apply, norm probe, solve, counters) works on it with m = G M0 + k rows in the reference's
 * order -- the G M0 observation rows (equation-major), then the k constraint rows (equation 0's first) --
 * and n = G N0 parameters.  z_scale / c_scale (G each) may be NULL (identity auxiliary). */
int glsgpu_mvrglm_create(int G, int64_t M0, int64_t N0, const double* Z0 /* M0 x N0 */, const double* Y /* M0 x G */,
                         const double* omega /* G x G */, const int64_t* roff, const int64_t* ridx,
                         const double* z_scale, const double* c_scale, int device, glsgpu_sur** out, int* bad_block);
/* mv_reduce: the thin QR Z0 = Q0 R0 on the device; R0 (N0 x N0) and Q0' Y (N0 x G), column-major.  R0 equals
 * the reference's up to the signs of its rows (a TSQR tree instead of one Householder sweep); the reduced
 * model is the same up to that orthogonal diagonal, which the GLS estimate does not see. */
int glsgpu_mv_reduce(int G, int64_t M0, int64_t N0, const double* Z0, const double* Y, double* R0, double* QtY,
                     int device);
/* sur_reduce (Remark-1 pre-pass): rotate every equation onto an orthonormal basis of range([X_1 ... X_G]).
 * Host X (M x n) and Y (M x G) in, q (the numerical rank, rank_tol as the reference's default 1e-10) and the
 * reduced X (q x n) and Y (q x G) out; X_red / Y_red must hold min(M, n) rows.  q == M: not reduced (copies).
 * basis (M x q) is optional.  Uses cuBLAS / cuSOLVER (dlopened) for the Gram, the eigensolver and the QR; the
 * basis equals the reference's up to an orthogonal q x q factor. */
int glsgpu_sur_reduce(int G, int64_t M, const int64_t* n_i, const double* X, const double* Y, double rank_tol,
                      int device, int64_t* q_out, double* X_red, double* Y_red, double* basis);
/* pcg_normal_equations(embed_sur(sur), nullptr, cfg, true_beta): the PCG-NE comparison solver on the handle's
 * SUR model (identity preconditioner).  b_out (n) required; w_out (m, the implied Sigma^-1 (y - X b)) and rows
 * optional; res->sigma_scale holds the G-norm probe.  SingularCovariance when Omega is not positive definite. */
int glsgpu_pcg_ne(glsgpu_sur* h, const glsgpu_pcg_config* cfg, const double* beta_true, double* b_out,
                  double* w_out, glsgpu_trace_row* rows, int64_t rows_cap, glsgpu_result* res);
/* m (rows of the reference's embedded GLM) and n of a handle. */
int glsgpu_model_dims(const glsgpu_sur* h, int64_t* m, int64_t* n);

/* Test / bench helpers (not part of the reference surface) ---------------------------------- */
/* Copy Q (M x n, ld M) and the concatenated R blocks to host. */
int glsgpu_get_factors(const glsgpu_sur* h, double* Q, double* R);
/* How the handle's blocks were factored: *method = 1 CholeskyQR2 on the FP64 tensor cores (csrc/cqr.cuh), 0 the
 * Householder TSQR (always when the environment says GLSGPU_QR=tsqr at creation); *fallbacks = factorisations of
 * this handle that failed CholeskyQR2's own orthogonality test and were redone by the TSQR. */
int glsgpu_factor_info(const glsgpu_sur* h, int* method, int* fallbacks);
/* Rows [row0, row0 + rows) of a rows_total x cols matrix of N(0,1) draws from the counter-based
 * Philox stream (seed, stream), into device memory with leading dimension ld: every row sharding of
 * the same matrix draws identical values. */
int glsgpu_synth_normal(double* dev, int64_t rows, int64_t cols, int64_t ld, int64_t row0, int64_t rows_total,
                        uint64_t seed, uint64_t stream, int device);
/* Device-side y_b = X_b beta_b + (Z Omega_half)_b for rows [row0, row0 + M) of M_total (Z: stream 3). */
int glsgpu_synth_response(int G, int64_t M, int64_t row0, int64_t M_total, const int64_t* n_i, const double* X_dev,
                          int64_t ldx, const double* beta, const double* omega_half, uint64_t seed, double* Y_dev,
                          int64_t ldy, int device);

#ifdef __cplusplus
}
#endif

#endif /* GLSGPU_H */
