/*
 * oracle/gls_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this library.  The product path (paper_2510_14471_b200, libglsgpu.so) never links
 * or calls it and fails loudly when its CUDA extension is missing.
 *
 * What it is: a plain-C restatement of the reference's PCG-Aug solver (Algorithm 3, the
 * "Recovery" variant) for SUR models with the per-block QR preconditioner and the Kronecker
 * covariance Sigma = Omega (x) I_M.  It follows the reference line by line; the only change is
 * that the dense block-diagonal X the reference materialises in embed_sur
 * (/root/reference/proj/src/structured.cpp:107-119) is never formed: every X apply /
 * X-transpose apply / Frobenius norm visits the blocks in the same column and row order, which
 * is bitwise identical because the off-block entries contribute exact +-0.
 *
 * Compile WITHOUT fused multiply-add contraction (-ffp-contract=off, no -march) so the
 * arithmetic matches the reference's default x86-64 SSE2 code generation.
 *
 * Parity pin: tests/test_oracle_vs_reference.py checks this restatement bitwise against the
 * reference itself, compiled from /root/reference by oracle/Makefile into oracle/_ref/.
 *
 * Layout (same as the reference): all matrices column-major.  X and Q are the concatenation of
 * the blocks [X_0 | X_1 | ... ] as one M x n matrix (block b owns columns [p0_b, p0_b + n_b));
 * R is the concatenation of the n_b x n_b blocks; Y and every m-vector are M x G column-major
 * (equation b owns rows [b*M, (b+1)*M) of the stacked vector).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Threads: the per-block loops (QR of each block, the Q / Q' / X / X' applies of each block), the
 * per-column Kronecker apply and the element-wise vector updates run in parallel over INDEPENDENT
 * outputs; every output keeps the reference's own sequential order, so the results are bitwise the
 * single-threaded ones.  The long dot products (vdot) stay sequential.  orc_set_threads(1) gives the
 * reference's single thread. */
static int orc_nthreads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
static int orc_tid(void) {
#ifdef _OPENMP
  return omp_get_thread_num();
#else
  return 0;
#endif
}
void orc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}
int orc_get_threads(void) { return orc_nthreads(); }
#define ORC_PAR _Pragma("omp parallel for schedule(static)")
#define ORC_PAR_DYN _Pragma("omp parallel for schedule(dynamic, 1)")

#define ORC_OK 0
#define ORC_DIMENSION_MISMATCH 1
#define ORC_RANK_DEFICIENT 2
#define ORC_SINGULAR_D 3
#define ORC_SINGULAR_TRIANGULAR 4
#define ORC_NO_MEMORY 12

/* Termination, same order as gls::Termination (proj/include/gls/glm.hpp:26). */
enum { T_CONVERGED = 0, T_BREAKDOWN = 1, T_STAGNATION = 2, T_MAXITER = 3, T_DIRECT = 4 };

/* Mirrors gls::PcgConfig (proj/include/gls/pcg.hpp:12-30). */
typedef struct {
  double tol_rel;
  int64_t max_iter;
  double breakdown_tol;
  int64_t stagnation_window;
  double growth_tol;
  int64_t growth_window;
  int64_t record_z_every;
} orc_config;

/* Mirrors gls::PcgTraceRow (proj/include/gls/pcg.hpp:32-39). */
typedef struct {
  int64_t iter;
  double c;
  double aug_residual_norm;
  double dual_feas_norm;
  double rmse;
  int64_t elapsed_ns;
} orc_trace_row;

/* Result: GlsSolution + PcgTrace scalars (proj/include/gls/glm.hpp:30-37, pcg.hpp:41-51). */
typedef struct {
  int64_t iterations;
  int32_t termination;
  int32_t w1_projected;
  int64_t breakdown_iteration; /* -1 when absent */
  double residual_seminorm;
  int64_t n_rows;              /* trace rows written (iterations + 1) */
  double sigma_scale;          /* operator_norm_probe result */
} orc_result;

/* ------------------------------------------------------------------ dense helpers
 * proj/src/dense_matrix.cpp:69-91,165-202 */

/* Summation mode of the long reductions (dot products, X'w / Q'r column dots).  0 = the reference's
 * sequential sums (default, bitwise the reference).  1 = pairwise (tree) sums -- a DIAGNOSTIC variant
 * in the accuracy class of the GPU's fixed-shape reduction trees, used to map the arithmetic envelope
 * of the iteration count; never used for parity claims against the reference. */
static int g_sum_mode = 0;
void orc_set_sum_mode(int mode) { g_sum_mode = mode; }

/* DIAGNOSTIC: per-iteration margins of the last orc_pcg_aug_sur call -- d / (uu sigma_scale) of the
 * breakdown test and c_next / c_best of the growth test -- to show how close a run was to a
 * roundoff-level stop.  Not part of the restatement's results. */
#define ORC_DIAG_MAX 100000
static double g_diag_d[ORC_DIAG_MAX], g_diag_g[ORC_DIAG_MAX];
static int64_t g_diag_n = 0;
int64_t orc_diag(double* d_ratio, double* growth, int64_t cap) {
  const int64_t n = g_diag_n < cap ? g_diag_n : cap;
  for (int64_t i = 0; i < n; ++i) {
    d_ratio[i] = g_diag_d[i];
    growth[i] = g_diag_g[i];
  }
  return n;
}

static double pairwise_dot(int64_t n, const double* a, const double* b) {
  if (n <= 32) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += a[i] * b[i];
    return acc;
  }
  const int64_t h = n / 2;
  return pairwise_dot(h, a, b) + pairwise_dot(n - h, a + h, b + h);
}

static double vdot(int64_t n, const double* a, const double* b) {
  if (g_sum_mode == 1) return pairwise_dot(n, a, b);
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc;
}
static double vnorm2(int64_t n, const double* a) { return sqrt(vdot(n, a, a)); }

/* y = A x (column-major rows x cols, leading dim ld), skipping x_j == 0 (dense_matrix.cpp:69-79) */
static void gemv(int64_t rows, int64_t cols, const double* a, int64_t ld, const double* x, double* y) {
  for (int64_t i = 0; i < rows; ++i) y[i] = 0.0;
  for (int64_t j = 0; j < cols; ++j) {
    const double xj = x[j];
    if (xj == 0.0) continue;
    const double* cj = a + j * ld;
    for (int64_t i = 0; i < rows; ++i) y[i] += cj[i] * xj;
  }
}
/* y = A' x, sequential dot per column (dense_matrix.cpp:81-91) */
static void gemv_t(int64_t rows, int64_t cols, const double* a, int64_t ld, const double* x, double* y) {
  if (g_sum_mode == 1) {
    for (int64_t j = 0; j < cols; ++j) y[j] = pairwise_dot(rows, a + j * ld, x);
    return;
  }
  for (int64_t j = 0; j < cols; ++j) {
    const double* cj = a + j * ld;
    double acc = 0.0;
    for (int64_t i = 0; i < rows; ++i) acc += cj[i] * x[i];
    y[j] = acc;
  }
}

/* ------------------------------------------------------------------ linalg
 * Householder QR: proj/src/linalg.cpp:24-117.  a is m x n (ld = m), overwritten with the packed
 * reflectors (unit-head convention, packed(k,k) = v0); beta[k] = 2/v'v; rdiag[k] = alpha. */
static void householder_factor(int64_t m, int64_t n, double* w, double* beta, double* rdiag) {
  for (int64_t k = 0; k < n; ++k) {
    double norm_x = 0.0;
    for (int64_t i = k; i < m; ++i) norm_x = hypot(norm_x, w[i + k * m]);
    if (norm_x == 0.0) {
      beta[k] = 0.0;
      rdiag[k] = 0.0;
      continue;
    }
    const double wkk = w[k + k * m];
    const double alpha = wkk >= 0.0 ? -norm_x : norm_x;
    const double v0 = wkk - alpha;
    beta[k] = -1.0 / (alpha * v0);
    w[k + k * m] = v0;
    for (int64_t i = k + 1; i < m; ++i) w[i + k * m] /= v0;
    const double beta_hat = beta[k] * v0 * v0;
    for (int64_t j = k + 1; j < n; ++j) {
      double s = w[k + j * m];
      for (int64_t i = k + 1; i < m; ++i) s += w[i + k * m] * w[i + j * m];
      s *= beta_hat;
      w[k + j * m] -= s;
      for (int64_t i = k + 1; i < m; ++i) w[i + j * m] -= s * w[i + k * m];
    }
    rdiag[k] = alpha;
  }
}

/* check_rank: proj/src/linalg.cpp:55-63 (kDefaultRankTol = 1e-10, linalg.hpp:10) */
static int check_rank(int64_t n, const double* rdiag, double rank_tol) {
  double max_d = 0.0, min_d = INFINITY;
  for (int64_t k = 0; k < n; ++k) {
    const double d = fabs(rdiag[k]);
    if (d > max_d) max_d = d;
    if (d < min_d) min_d = d;
  }
  if (max_d == 0.0 || min_d <= rank_tol * max_d) return ORC_RANK_DEFICIENT;
  return ORC_OK;
}

/* form_q_columns(f, 0, n): proj/src/linalg.cpp:77-95; q is m x n (ld = ldq) */
static void form_q(int64_t m, int64_t n, const double* packed, const double* beta, double* q, int64_t ldq) {
  for (int64_t j = 0; j < n; ++j) {
    for (int64_t i = 0; i < m; ++i) q[i + j * ldq] = 0.0;
    q[j + j * ldq] = 1.0;
  }
  for (int64_t k = n; k-- > 0;) {
    if (beta[k] == 0.0) continue;
    const double v0 = packed[k + k * m];
    const double beta_hat = beta[k] * v0 * v0;
    for (int64_t j = 0; j < n; ++j) {
      double* qj = q + j * ldq;
      double s = qj[k];
      for (int64_t i = k + 1; i < m; ++i) s += packed[i + k * m] * qj[i];
      s *= beta_hat;
      qj[k] -= s;
      for (int64_t i = k + 1; i < m; ++i) qj[i] -= s * packed[i + k * m];
    }
  }
}

/* qr_thin: proj/src/linalg.cpp:110-117.  a: m x n (ld = lda), q: m x n (ld = ldq), r: n x n. */
int orc_qr_thin(int64_t m, int64_t n, const double* a, int64_t lda, double scale, double* q, int64_t ldq,
                double* r) {
  if (m < n || n == 0) return ORC_DIMENSION_MISMATCH;
  double* w = (double*)malloc(sizeof(double) * (size_t)(m * n));
  double* beta = (double*)malloc(sizeof(double) * (size_t)n);
  double* rdiag = (double*)malloc(sizeof(double) * (size_t)n);
  if (!w || !beta || !rdiag) { free(w); free(beta); free(rdiag); return ORC_NO_MEMORY; }
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) w[i + j * m] = a[i + j * lda] * scale; /* DenseMatrix *= w */
  householder_factor(m, n, w, beta, rdiag);
  int st = check_rank(n, rdiag, 1e-10);
  if (st == ORC_OK) {
    form_q(m, n, w, beta, q, ldq);
    /* extract_r: proj/src/linalg.cpp:65-73 */
    for (int64_t j = 0; j < n; ++j) {
      for (int64_t i = 0; i < n; ++i) r[i + j * n] = 0.0;
      for (int64_t i = 0; i < j; ++i) r[i + j * n] = w[i + j * m];
      r[j + j * n] = rdiag[j];
    }
  }
  free(w); free(beta); free(rdiag);
  return st;
}

/* tri_solve(R, b) with R upper triangular: proj/src/linalg.cpp:119-145 (Left side). */
static int tri_solve(int64_t n, const double* r, double* x, int transpose) {
  for (int64_t i = 0; i < n; ++i)
    if (r[i + i * n] == 0.0) return ORC_SINGULAR_TRIANGULAR;
  if (!transpose) {
    for (int64_t i = n; i-- > 0;) {
      double s = x[i];
      for (int64_t j = i + 1; j < n; ++j) s -= r[i + j * n] * x[j];
      x[i] = s / r[i + i * n];
    }
  } else {
    for (int64_t i = 0; i < n; ++i) {
      double s = x[i];
      for (int64_t j = 0; j < i; ++j) s -= r[j + i * n] * x[j];
      x[i] = s / r[i + i * n];
    }
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------ the SUR operator
 * SurPreconditioner / BlockQrPreconditioner: proj/src/structured.cpp:282-363,416-453. */
typedef struct {
  int G;
  int64_t M;
  int64_t n; /* total params */
  const int64_t* nb;
  int64_t* p0;  /* first parameter index per block */
  int64_t* r0;  /* offset of R_b in the concatenated R */
  double* Q;    /* M x n */
  double* R;    /* concatenated */
  double* wts;  /* 1/sqrt(block_scale) */
  double* local; /* per-thread scratch: nthr x M */
  double* tvec;  /* per-thread scratch: nthr x nmax */
  int nthr;
  int64_t nmax;
} orc_sur;

static void orc_sur_free(orc_sur* s) {
  if (!s) return;
  free(s->p0); free(s->r0); free(s->Q); free(s->R); free(s->wts); free(s->local); free(s->tvec);
  free(s);
}

static int64_t total_params(int G, const int64_t* nb) {
  int64_t n = 0;
  for (int b = 0; b < G; ++b) n += nb[b];
  return n;
}

/* Build the operator: per block, qr_thin of w * X_b (structured.cpp:427-450). bad_block gets the
 * failing block index for RankDeficient / SingularD. */
static int orc_sur_build(int G, int64_t M, const int64_t* nb, const double* X, const double* scale,
                         orc_sur** out, int* bad_block) {
  *out = NULL;
  if (G < 1) return ORC_DIMENSION_MISMATCH;
  orc_sur* s = (orc_sur*)calloc(1, sizeof(orc_sur));
  if (!s) return ORC_NO_MEMORY;
  s->G = G; s->M = M; s->nb = nb; s->n = total_params(G, nb);
  int64_t rtot = 0, nmax = 0;
  for (int b = 0; b < G; ++b) { rtot += nb[b] * nb[b]; if (nb[b] > nmax) nmax = nb[b]; }
  s->p0 = (int64_t*)malloc(sizeof(int64_t) * G);
  s->r0 = (int64_t*)malloc(sizeof(int64_t) * G);
  s->Q = (double*)malloc(sizeof(double) * (size_t)(M * s->n));
  s->R = (double*)malloc(sizeof(double) * (size_t)(rtot > 0 ? rtot : 1));
  s->wts = (double*)malloc(sizeof(double) * G);
  s->nthr = orc_nthreads();
  s->nmax = nmax > 0 ? nmax : 1;
  s->local = (double*)malloc(sizeof(double) * (size_t)M * (size_t)s->nthr);
  s->tvec = (double*)malloc(sizeof(double) * (size_t)s->nmax * (size_t)s->nthr);
  if (!s->p0 || !s->r0 || !s->Q || !s->R || !s->wts || !s->local || !s->tvec) { orc_sur_free(s); return ORC_NO_MEMORY; }
  int64_t p = 0, r = 0;
  for (int b = 0; b < G; ++b) {
    if (scale && scale[b] <= 0.0) { if (bad_block) *bad_block = b; orc_sur_free(s); return ORC_SINGULAR_D; }
    const double w = scale ? 1.0 / sqrt(scale[b]) : 1.0 / sqrt(1.0);
    s->wts[b] = w;
    s->p0[b] = p; s->r0[b] = r;
    p += nb[b]; r += nb[b] * nb[b];
  }
  /* the blocks' QRs are independent; the first failing block (in block order) is reported, as the
   * reference's sequential loop would */
  int* bst = (int*)malloc(sizeof(int) * (size_t)G);
  if (!bst) { orc_sur_free(s); return ORC_NO_MEMORY; }
  ORC_PAR_DYN
  for (int b = 0; b < G; ++b)
    bst[b] = orc_qr_thin(M, nb[b], X + s->p0[b] * M, M, s->wts[b], s->Q + s->p0[b] * M, M, s->R + s->r0[b]);
  for (int b = 0; b < G; ++b)
    if (bst[b] != ORC_OK) {
      const int st = bst[b];
      if (bad_block) *bad_block = b;
      free(bst);
      orc_sur_free(s);
      return st;
    }
  free(bst);
  *out = s;
  return ORC_OK;
}

/* pi_impl: proj/src/structured.cpp:307-317 */
static void sur_pi(const orc_sur* s, const double* xi, double* out) {
  const int64_t M = s->M;
  ORC_PAR_DYN
  for (int b = 0; b < s->G; ++b) {
    const double w = s->wts[b];
    const int64_t nbb = s->nb[b];
    const double* Qb = s->Q + s->p0[b] * M;
    double* local = s->local + (size_t)orc_tid() * (size_t)M;
    double* tvec = s->tvec + (size_t)orc_tid() * (size_t)s->nmax;
    for (int64_t i = 0; i < M; ++i) local[i] = xi[b * M + i] * w;             /* gather */
    gemv_t(M, nbb, Qb, M, local, tvec);                                         /* Q' local */
    for (int64_t i = 0; i < M; ++i) out[b * M + i] = 0.0;
    /* proj = Q t, then local -= proj: do it in the reference's order (apply then subtract) */
    double* proj = out + b * M; /* reuse output slot as proj scratch */
    gemv(M, nbb, Qb, M, tvec, proj);
    for (int64_t i = 0; i < M; ++i) local[i] -= proj[i];
    for (int64_t i = 0; i < M; ++i) out[b * M + i] = local[i] * w;              /* scatter */
  }
}

/* xstar_t_impl: proj/src/structured.cpp:319-328 */
static int sur_xstar_t(const orc_sur* s, const double* xi, double* out) {
  const int64_t M = s->M;
  int st_all = ORC_OK;
  ORC_PAR_DYN
  for (int b = 0; b < s->G; ++b) {
    const double w = s->wts[b];
    const int64_t nbb = s->nb[b];
    double* local = s->local + (size_t)orc_tid() * (size_t)M;
    for (int64_t i = 0; i < M; ++i) local[i] = xi[b * M + i] * w;
    gemv_t(M, nbb, s->Q + s->p0[b] * M, M, local, out + s->p0[b]);
    int st = tri_solve(nbb, s->R + s->r0[b], out + s->p0[b], 0);
    if (st) {
#pragma omp atomic write
      st_all = st;
    }
  }
  return st_all;
}

/* xstar_impl: proj/src/structured.cpp:330-340 */
static int sur_xstar(const orc_sur* s, const double* v, double* out) {
  const int64_t M = s->M;
  int st_all = ORC_OK;
  ORC_PAR_DYN
  for (int b = 0; b < s->G; ++b) {
    const double w = s->wts[b];
    const int64_t nbb = s->nb[b];
    double* vi = s->tvec + (size_t)orc_tid() * (size_t)s->nmax;
    double* local = s->local + (size_t)orc_tid() * (size_t)M;
    memcpy(vi, v + s->p0[b], sizeof(double) * (size_t)nbb);
    int st = tri_solve(nbb, s->R + s->r0[b], vi, 1);
    if (st) {
#pragma omp atomic write
      st_all = st;
      continue;
    }
    gemv(M, nbb, s->Q + s->p0[b] * M, M, vi, local);
    for (int64_t i = 0; i < M; ++i) out[b * M + i] = local[i] * w;
  }
  return st_all;
}

/* ------------------------------------------------------------------ structured X applies
 * The reference applies the dense embed_sur X (structured.cpp:107-119) with
 * DenseMatrix::apply / apply_transpose (dense_matrix.cpp:69-91).  Per block, same order. */
static void x_apply(int G, int64_t M, const int64_t* nb, const double* X, const double* v, double* y) {
  int64_t* p0 = (int64_t*)malloc(sizeof(int64_t) * (size_t)G);
  int64_t p = 0;
  for (int b = 0; b < G; ++b) { p0[b] = p; p += nb[b]; }
  ORC_PAR_DYN
  for (int b = 0; b < G; ++b) gemv(M, nb[b], X + p0[b] * M, M, v + p0[b], y + b * M);
  free(p0);
}
static void x_apply_t(int G, int64_t M, const int64_t* nb, const double* X, const double* w, double* out) {
  int64_t* p0 = (int64_t*)malloc(sizeof(int64_t) * (size_t)G);
  int64_t p = 0;
  for (int b = 0; b < G; ++b) { p0[b] = p; p += nb[b]; }
  ORC_PAR_DYN
  for (int b = 0; b < G; ++b) gemv_t(M, nb[b], X + p0[b] * M, M, w + b * M, out + p0[b]);
  free(p0);
}
static double x_frobenius(int G, int64_t M, const int64_t* nb, const double* X) {
  /* DenseMatrix::frobenius_norm (dense_matrix.cpp:93-97): storage order, off-block zeros add +0 */
  const int64_t n = total_params(G, nb);
  double acc = 0.0;
  for (int64_t k = 0; k < M * n; ++k) acc += X[k] * X[k];
  (void)G;
  return sqrt(acc);
}

/* ------------------------------------------------------------------ Kronecker Sigma apply
 * SymmetricOperator::apply Kron branch (proj/src/operators.cpp:45-50): vec(reshape(x,M,G) * core)
 * with operator* (dense_matrix.cpp:125-139): j -> p -> i, skipping core(p,j) == 0. */
void orc_kron_apply(int G, int64_t M, const double* omega, const double* x, double* out) {
  /* row tiles are independent; inside a tile the j -> p -> i order of operator* is kept, so every
   * output is the same p-ascending sum as the reference's */
  const int64_t TR = 512;
  const int64_t ntile = (M + TR - 1) / TR;
  ORC_PAR_DYN
  for (int64_t t = 0; t < ntile; ++t) {
    const int64_t i0 = t * TR, i1 = (i0 + TR < M) ? i0 + TR : M;
    for (int j = 0; j < G; ++j) {
      double* cj = out + (int64_t)j * M;
      for (int64_t i = i0; i < i1; ++i) cj[i] = 0.0;
      for (int p = 0; p < G; ++p) {
        const double bpj = omega[p + (int64_t)j * G];
        if (bpj == 0.0) continue;
        const double* ap = x + (int64_t)p * M;
        for (int64_t i = i0; i < i1; ++i) cj[i] += ap[i] * bpj;
      }
    }
  }
}

/* operator_norm_probe: proj/src/pcg.cpp:233-244 */
double orc_norm_probe(int G, int64_t M, const double* omega, int64_t iters) {
  const int64_t m = M * G;
  double* v = (double*)malloc(sizeof(double) * (size_t)m);
  double* t = (double*)malloc(sizeof(double) * (size_t)m);
  for (int64_t i = 0; i < m; ++i) v[i] = 1.0 / sqrt((double)m);
  double nrm = 0.0;
  for (int64_t it = 0; it < iters; ++it) {
    orc_kron_apply(G, M, omega, v, t);
    memcpy(v, t, sizeof(double) * (size_t)m);
    nrm = vnorm2(m, v);
    if (nrm == 0.0) { free(v); free(t); return 0.0; }
    for (int64_t i = 0; i < m; ++i) v[i] /= nrm;
  }
  free(v); free(t);
  return nrm;
}

/* ------------------------------------------------------------------ exported operator probes */
int orc_sur_setup(int G, int64_t M, const int64_t* nb, const double* X, const double* scale, double* Q_out,
                  double* R_out, int* bad_block) {
  orc_sur* s = NULL;
  int st = orc_sur_build(G, M, nb, X, scale, &s, bad_block);
  if (st) return st;
  memcpy(Q_out, s->Q, sizeof(double) * (size_t)(M * s->n));
  int64_t rtot = 0;
  for (int b = 0; b < G; ++b) rtot += nb[b] * nb[b];
  memcpy(R_out, s->R, sizeof(double) * (size_t)rtot);
  orc_sur_free(s);
  return ORC_OK;
}

/* kind: 0 = apply_pi (m -> m), 1 = apply_xstar_t (m -> n), 2 = apply_xstar (n -> m) */
int orc_sur_apply(int G, int64_t M, const int64_t* nb, const double* X, const double* scale, int kind,
                  const double* in, double* out) {
  orc_sur* s = NULL;
  int bad = -1;
  int st = orc_sur_build(G, M, nb, X, scale, &s, &bad);
  if (st) return st;
  if (kind == 0) sur_pi(s, in, out);
  else if (kind == 1) st = sur_xstar_t(s, in, out);
  else st = sur_xstar(s, in, out);
  orc_sur_free(s);
  return st;
}

static int64_t now_ns(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (int64_t)ts.tv_sec * 1000000000LL + ts.tv_nsec;
}

/* ------------------------------------------------------------------ the model behind run_aug
 * run_aug only touches the GLM through X, X', |X|_F, Sigma and operator_norm_probe(Sigma), and the
 * preconditioner through pi / xstar_t / xstar: these hooks restate them per model class. */
typedef struct {
  int64_t m, n;
  const void* ctx;
  void (*x_apply)(const void*, const double* v, double* y);
  void (*x_apply_t)(const void*, const double* w, double* out);
  double (*x_frob)(const void*);
  void (*sigma)(const void*, const double* x, double* out);
  void (*pi)(const void*, const double* xi, double* out);
  int (*xstar_t)(const void*, const double* xi, double* out);
  int (*xstar)(const void*, const double* v, double* out);
} orc_model;

/* operator_norm_probe(glm.sigma) (pcg.cpp:233-244) through the model's Sigma hook */
static double model_norm_probe(const orc_model* mo, int64_t iters) {
  const int64_t m = mo->m;
  double* v = (double*)malloc(sizeof(double) * (size_t)m);
  double* t = (double*)malloc(sizeof(double) * (size_t)m);
  for (int64_t i = 0; i < m; ++i) v[i] = 1.0 / sqrt((double)m);
  double nrm = 0.0;
  for (int64_t it = 0; it < iters; ++it) {
    mo->sigma(mo->ctx, v, t);
    memcpy(v, t, sizeof(double) * (size_t)m);
    nrm = vnorm2(m, v);
    if (nrm == 0.0) break;
    for (int64_t i = 0; i < m; ++i) v[i] /= nrm;
  }
  free(v); free(t);
  return nrm;
}

/* ------------------------------------------------------------------ run_aug, Recovery variant
 * proj/src/pcg.cpp:36-229 (entered through pcg_aug, pcg.cpp:346-350) on a model (hooks above).
 *
 * w1 / z1 may be NULL (zeros); beta_true may be NULL (rmse = NaN).  rows may be NULL (trace not
 * returned); otherwise it must hold max_iter + 1 rows.  b_out: n, w_out: m (may be NULL). */
static int run_aug(const orc_model* mo, const double* Y, const double* w1, const double* z1,
                   const orc_config* cfg, const double* beta_true, double* b_out, double* w_out,
                   orc_trace_row* rows, int64_t rows_cap, orc_result* res) {
  const int64_t m = mo->m, n = mo->n;
  const void* s = mo->ctx;
  int st = ORC_OK;
  if (m < n) return ORC_DIMENSION_MISMATCH; /* make_glm: m > n (glm.cpp:10-16) */

  const int64_t max_iter = cfg->max_iter ? cfg->max_iter : (m - n + 1); /* pcg.cpp:34,46-47 */
  const int64_t stride = cfg->record_z_every ? cfg->record_z_every : 1;
  const double sigma_scale = model_norm_probe(mo, 12);
  const int64_t start = now_ns();

  size_t mb = sizeof(double) * (size_t)m, nbytes = sizeof(double) * (size_t)(n > 0 ? n : 1);
  double *w = malloc(mb), *sw = malloc(mb), *r = malloc(mb), *pr = malloc(mb), *u = malloc(mb), *su = malloc(mb),
         *xv = malloc(mb), *tmp = malloc(mb), *w_best = malloc(mb), *sw_best = malloc(mb);
  double *z = malloc(nbytes), *v = malloc(nbytes), *xtw = malloc(nbytes), *est = malloc(nbytes),
         *xr = malloc(nbytes);
  if (!w || !sw || !r || !pr || !u || !su || !xv || !tmp || !w_best || !sw_best || !z || !v || !xtw || !est || !xr) {
    st = ORC_NO_MEMORY;
    goto done;
  }
  int64_t nrows = 0;
  res->w1_projected = 0;
  res->breakdown_iteration = -1;
  res->sigma_scale = sigma_scale;

  /* Enforce X'w1 = 0 (pcg.cpp:55-66) */
  if (w1) memcpy(w, w1, mb); else memset(w, 0, mb);
  {
    mo->x_apply_t(s, w, xtw);
    const double feas = vnorm2(n, xtw);
    const double sc = mo->x_frob(s) * vnorm2(m, w);
    if (feas > 1e-14 * sc && feas > 0.0) {
      st = mo->xstar(s, xtw, tmp);
      if (st) goto done;
      ORC_PAR
      for (int64_t i = 0; i < m; ++i) w[i] -= tmp[i];
      res->w1_projected = 1;
    }
  }
  if (z1) memcpy(z, z1, nbytes); else memset(z, 0, nbytes);
  mo->sigma(s, w, sw);                                                  /* sw = Sigma w */
  mo->x_apply(s, z, xv);
  ORC_PAR
  for (int64_t i = 0; i < m; ++i) r[i] = (sw[i] + xv[i]) - Y[i];         /* sub(add(sw, Xz), y) */
  mo->pi(s, r, pr);
  double c = vdot(m, r, pr);
  if (c < 0.0) c = 0.0;                                                  /* max(dot, 0) */
  const double c1 = c;
  const double threshold = cfg->tol_rel * cfg->tol_rel * c1;

  /* c_floor (pcg.cpp:79-86) */
  const double kEpsC = DBL_EPSILON;
  double pi_gain = 0.0;
#define C_FLOOR(rn2, prn)                                                          \
  ((rn2) > 0.0 ? (pi_gain = fmax(pi_gain, (prn) / sqrt(rn2))) : 0.0,               \
   16.0 * kEpsC * fmax(pi_gain, 1e-3) * (rn2))
  (void)C_FLOOR(vdot(m, r, r), vnorm2(m, pr));

  memcpy(u, pr, mb);
  st = mo->xstar_t(s, r, v);
  if (st) goto done;

  /* recover(sw) = X*'(y - sw) and push_row (pcg.cpp:96-116) */
#define RECOVER(swsel, outv)                                           \
  do {                                                                 \
    ORC_PAR \
    for (int64_t i_ = 0; i_ < m; ++i_) tmp[i_] = Y[i_] - (swsel)[i_];  \
    st = mo->xstar_t(s, tmp, (outv));                                  \
    if (st) goto done;                                                 \
  } while (0)
#define PUSH_ROW(iter_, cval_, sampled_)                                                       \
  do {                                                                                         \
    if (rows && nrows < rows_cap) {                                                            \
      orc_trace_row* row_ = &rows[nrows];                                                      \
      row_->iter = (iter_);                                                                    \
      row_->c = (cval_);                                                                       \
      mo->x_apply(s, est, tmp);                                                                \
      ORC_PAR \
      for (int64_t i_ = 0; i_ < m; ++i_) tmp[i_] = Y[i_] - (sw[i_] + tmp[i_]);                 \
      row_->aug_residual_norm = vnorm2(m, tmp);                                                \
      mo->x_apply_t(s, w, xtw);                                                                \
      row_->dual_feas_norm = vnorm2(n, xtw);                                                   \
      if ((sampled_) && beta_true) {                                                           \
        double acc_ = 0.0;                                                                     \
        for (int64_t k_ = 0; k_ < n; ++k_) { const double d_ = est[k_] - beta_true[k_]; acc_ += d_ * d_; } \
        row_->rmse = sqrt(acc_ / (double)n);                                                   \
      } else {                                                                                 \
        row_->rmse = NAN;                                                                      \
      }                                                                                        \
      row_->elapsed_ns = now_ns() - start;                                                     \
    }                                                                                          \
    ++nrows;                                                                                   \
  } while (0)

  RECOVER(sw, est);
  PUSH_ROW(0, c, 1);

  memcpy(w_best, w, mb);
  memcpy(sw_best, sw, mb);
  double c_best = c;
  int64_t best_iter = 0, stagnant = 0, done_it = 0;
  int term = T_MAXITER;

  g_diag_n = 0;
  if (c1 == 0.0) {
    term = T_CONVERGED;
  } else {
    for (int64_t i = 1; i <= max_iter; ++i) {
      mo->sigma(s, u, su);                                              /* su = Sigma u */
      const double d = vdot(m, u, su);
      if (i - 1 < ORC_DIAG_MAX) {
        g_diag_d[i - 1] = fabs(d) / (vdot(m, u, u) * sigma_scale);
        g_diag_g[i - 1] = 0.0;
        g_diag_n = i;
      }
      if (fabs(d) <= cfg->breakdown_tol * vdot(m, u, u) * sigma_scale) {
        term = T_BREAKDOWN;
        res->breakdown_iteration = i;
        break;
      }
      const double lambda = c / d;
      ORC_PAR
      for (int64_t k = 0; k < m; ++k) w[k] += -lambda * u[k];          /* axpy(-lambda, u, w) */
      ORC_PAR
      for (int64_t k = 0; k < m; ++k) sw[k] += -lambda * su[k];        /* axpy(-lambda, su, sw) */
      mo->x_apply(s, v, xv);
      ORC_PAR
      for (int64_t k = 0; k < m; ++k) r[k] -= lambda * (su[k] + xv[k]);
      mo->pi(s, r, pr);
      double c_next = vdot(m, r, pr);
      done_it = i;

      const int sampled = (i % stride == 0) || c_next <= threshold || i == max_iter;
      RECOVER(sw, est);
      PUSH_ROW(i, c_next, sampled);

      const double floor_c = C_FLOOR(vdot(m, r, r), vnorm2(m, pr));
      const int exhausted = fabs(c_next) <= floor_c / 64.0 || (fabs(c_next) <= floor_c && c_next <= 1e-6 * c);
      if (c_next < 0.0 && fabs(c_next) > floor_c) {
        term = T_BREAKDOWN;
        res->breakdown_iteration = i;
        break;
      }
      if (c_next < 0.0) c_next = 0.0;
      if (i - 1 < ORC_DIAG_MAX) g_diag_g[i - 1] = c_best > 0.0 ? c_next / c_best : 0.0;
      if (c_next < c_best) {
        c_best = c_next;
        memcpy(w_best, w, mb);
        memcpy(sw_best, sw, mb);
        best_iter = i;
      }
      if (c_next <= threshold || exhausted) {
        term = T_CONVERGED;
        break;
      }
      if (fabs(c_next - c) <= 1e-15 * c) {
        if (++stagnant >= cfg->stagnation_window) {
          term = T_STAGNATION;
          break;
        }
      } else {
        stagnant = 0;
      }
      if (c_next > cfg->growth_tol * c_best && i - best_iter >= cfg->growth_window) {
        term = T_BREAKDOWN;
        res->breakdown_iteration = i;
        break;
      }
      const double mu = c_next / c;
      c = c_next;
      st = mo->xstar_t(s, r, xr);
      if (st) goto done;
      for (int64_t k = 0; k < n; ++k) v[k] = xr[k] + mu * v[k];
      ORC_PAR
      for (int64_t k = 0; k < m; ++k) u[k] = pr[k] + mu * u[k];
    }
  }

  {
    const int keep_last = term == T_CONVERGED;
    const double* w_sel = keep_last ? w : w_best;
    const double* sw_sel = keep_last ? sw : sw_best;
    if (w_out) memcpy(w_out, w_sel, mb);
    RECOVER(sw_sel, b_out);
    res->iterations = done_it;
    res->termination = term;
    res->residual_seminorm = keep_last ? c : c_best;
    res->n_rows = nrows;
  }
#undef C_FLOOR
#undef RECOVER
#undef PUSH_ROW

done:
  free(w); free(sw); free(r); free(pr); free(u); free(su); free(xv); free(tmp); free(w_best); free(sw_best);
  free(z); free(v); free(xtw); free(est); free(xr);
  return st;
}

/* ------------------------------------------------------------------ SUR: embed_sur + sur_preconditioner */
typedef struct {
  int G;
  int64_t M;
  const int64_t* nb;
  const double* X;
  const double* omega;
  const orc_sur* op;
} sur_model;

static void sur_h_x(const void* c, const double* v, double* y) {
  const sur_model* q = (const sur_model*)c;
  x_apply(q->G, q->M, q->nb, q->X, v, y);
}
static void sur_h_xt(const void* c, const double* w, double* out) {
  const sur_model* q = (const sur_model*)c;
  x_apply_t(q->G, q->M, q->nb, q->X, w, out);
}
static double sur_h_frob(const void* c) {
  const sur_model* q = (const sur_model*)c;
  return x_frobenius(q->G, q->M, q->nb, q->X);
}
static void sur_h_sigma(const void* c, const double* x, double* out) {
  const sur_model* q = (const sur_model*)c;
  orc_kron_apply(q->G, q->M, q->omega, x, out);
}
static void sur_h_pi(const void* c, const double* xi, double* out) { sur_pi(((const sur_model*)c)->op, xi, out); }
static int sur_h_xt_star(const void* c, const double* xi, double* out) {
  return sur_xstar_t(((const sur_model*)c)->op, xi, out);
}
static int sur_h_xstar(const void* c, const double* v, double* out) { return sur_xstar(((const sur_model*)c)->op, v, out); }

/* pcg_aug(embed_sur(sur), *sur_preconditioner(sur[, block_scale]), w1, z1, cfg, beta_true) */
int orc_pcg_aug_sur(int G, int64_t M, const int64_t* nb, const double* X, const double* Y, const double* omega,
                    const double* scale, const double* w1, const double* z1, const orc_config* cfg,
                    const double* beta_true, double* b_out, double* w_out, orc_trace_row* rows,
                    int64_t rows_cap, orc_result* res, int* bad_block) {
  orc_sur* s = NULL;
  int st = orc_sur_build(G, M, nb, X, scale, &s, bad_block);
  if (st) return st;
  sur_model q = {G, M, nb, X, omega, s};
  orc_model mo = {M * G, s->n, &q, sur_h_x, sur_h_xt, sur_h_frob, sur_h_sigma, sur_h_pi, sur_h_xt_star, sur_h_xstar};
  st = run_aug(&mo, Y, w1, z1, cfg, beta_true, b_out, w_out, rows, rows_cap, res);
  orc_sur_free(s);
  return st;
}

/* ------------------------------------------------------------------ MVRGLM
 * The multivariate model with exclusion restrictions (proj/include/gls/structured.hpp:37-52):
 *   glm  = embed_mvrglm(mv)          (structured.cpp:77-95): X = [I_G (x) Z0 ; C], y = [vec Y ; 0_k],
 *                                     Sigma = diag(Omega0 (x) I_M0, 0_k) (SymmetricOperator Padded)
 *   op   = mvrglm_preconditioner(mv[, z_scale, c_scale])  (structured.cpp:365-414)
 * The embedded row order is the reference's: rows [i M0, (i + 1) M0) are equation i's observations,
 * then the k constraint rows, equation 0's first.  Restrictions come as CSR: equation i restricts the
 * parameters ridx[roff[i] .. roff[i + 1]) (strictly increasing, < N0).  Nothing dense is formed: every
 * X / X' / |X|_F / Sigma apply visits the non-zeros in the dense routine's order (off-pattern entries
 * add exact +-0, as for SUR). */
typedef struct {
  int G;
  int64_t M0, N0, m, k, n;
  const double* Z0;     /* M0 x N0 */
  const double* omega;  /* G x G */
  const int64_t* roff;
  const int64_t* ridx;
  double* wz;           /* 1/sqrt(z_scale_i) */
  double* wc;           /* 1/sqrt(c_scale_i) */
  int64_t* qoff;        /* Q_i: (M0 + k_i) x N0 at qoff[i] */
  double* Q;
  double* R;            /* G x (N0 x N0) */
  double* local;
  double* tvec;
} orc_mv;

static void orc_mv_free(orc_mv* s) {
  if (!s) return;
  free(s->wz); free(s->wc); free(s->qoff); free(s->Q); free(s->R); free(s->local); free(s->tvec);
  free(s);
}

/* MvRglmPreconditioner ctor (structured.cpp:367-411): per equation, qr_thin of the stacked
 * [Z0 w_z ; C_i w_c] with C_i(r, restr_i[r]) = 1 */
static int orc_mv_build(int G, int64_t M0, int64_t N0, const double* Z0, const double* omega, const int64_t* roff,
                        const int64_t* ridx, const double* z_scale, const double* c_scale, orc_mv** out,
                        int* bad_block) {
  *out = NULL;
  if (G < 1 || M0 < N0 || N0 < 1) return ORC_DIMENSION_MISMATCH; /* make_mvrglm: Z0 tall */
  for (int i = 0; i < G; ++i)
    for (int64_t q = roff[i]; q < roff[i + 1]; ++q)
      if (ridx[q] < 0 || ridx[q] >= N0 || (q > roff[i] && ridx[q] <= ridx[q - 1])) return ORC_DIMENSION_MISMATCH;
  orc_mv* s = (orc_mv*)calloc(1, sizeof(orc_mv));
  if (!s) return ORC_NO_MEMORY;
  s->G = G; s->M0 = M0; s->N0 = N0; s->Z0 = Z0; s->omega = omega; s->roff = roff; s->ridx = ridx;
  s->k = roff[G];
  s->m = (int64_t)G * M0;
  s->n = (int64_t)G * N0;
  int64_t kmax = 0, qtot = 0;
  for (int i = 0; i < G; ++i) {
    const int64_t ki = roff[i + 1] - roff[i];
    if (ki > kmax) kmax = ki;
    qtot += (M0 + ki) * N0;
  }
  s->wz = (double*)malloc(sizeof(double) * G);
  s->wc = (double*)malloc(sizeof(double) * G);
  s->qoff = (int64_t*)malloc(sizeof(int64_t) * G);
  s->Q = (double*)malloc(sizeof(double) * (size_t)qtot);
  s->R = (double*)malloc(sizeof(double) * (size_t)(G * N0 * N0));
  s->local = (double*)malloc(sizeof(double) * (size_t)(M0 + kmax));
  s->tvec = (double*)malloc(sizeof(double) * (size_t)N0);
  double* stacked = (double*)malloc(sizeof(double) * (size_t)((M0 + kmax) * N0));
  if (!s->wz || !s->wc || !s->qoff || !s->Q || !s->R || !s->local || !s->tvec || !stacked) {
    free(stacked); orc_mv_free(s); return ORC_NO_MEMORY;
  }
  for (int i = 0; i < G; ++i) {
    const double zs = z_scale ? z_scale[i] : 1.0, cs = c_scale ? c_scale[i] : 1.0;
    if (zs <= 0.0 || cs <= 0.0) { if (bad_block) *bad_block = i; free(stacked); orc_mv_free(s); return ORC_SINGULAR_D; }
  }
  int64_t q0 = 0;
  for (int i = 0; i < G; ++i) {
    const int64_t ki = roff[i + 1] - roff[i], rows = M0 + ki;
    const double wz = 1.0 / sqrt(z_scale ? z_scale[i] : 1.0);
    const double wc = 1.0 / sqrt(c_scale ? c_scale[i] : 1.0);
    s->wz[i] = wz; s->wc[i] = wc;
    memset(stacked, 0, sizeof(double) * (size_t)(rows * N0));
    for (int64_t j = 0; j < N0; ++j)
      for (int64_t r = 0; r < M0; ++r) stacked[r + j * rows] = Z0[r + j * M0] * wz;
    for (int64_t r = 0; r < ki; ++r) stacked[M0 + r + ridx[roff[i] + r] * rows] = wc;
    s->qoff[i] = q0;
    int st = orc_qr_thin(rows, N0, stacked, rows, 1.0, s->Q + q0, rows, s->R + (int64_t)i * N0 * N0);
    if (st != ORC_OK) { if (bad_block) *bad_block = i; free(stacked); orc_mv_free(s); return st; }
    q0 += rows * N0;
  }
  free(stacked);
  *out = s;
  return ORC_OK;
}

/* embedded row of local row r of equation i (Block::row_index, structured.cpp:392-400) */
static int64_t mv_row(const orc_mv* s, int i, int64_t r) {
  return r < s->M0 ? (int64_t)i * s->M0 + r : s->m + s->roff[i] + (r - s->M0);
}
static double mv_isd(const orc_mv* s, int i, int64_t r) { return r < s->M0 ? s->wz[i] : s->wc[i]; }

/* BlockQrPreconditioner::pi_impl / xstar_t_impl / xstar_impl (structured.cpp:307-340) */
static void mv_pi(const void* c, const double* xi, double* out) {
  const orc_mv* s = (const orc_mv*)c;
  const int64_t N0 = s->N0;
  for (int64_t i = 0; i < s->m + s->k; ++i) out[i] = 0.0;
  double* proj = (double*)malloc(sizeof(double) * (size_t)(s->M0 + s->k + 1));
  for (int i = 0; i < s->G; ++i) {
    const int64_t rows = s->M0 + (s->roff[i + 1] - s->roff[i]);
    const double* Qi = s->Q + s->qoff[i];
    for (int64_t r = 0; r < rows; ++r) s->local[r] = xi[mv_row(s, i, r)] * mv_isd(s, i, r);
    gemv_t(rows, N0, Qi, rows, s->local, s->tvec);
    gemv(rows, N0, Qi, rows, s->tvec, proj);
    for (int64_t r = 0; r < rows; ++r) s->local[r] -= proj[r];
    for (int64_t r = 0; r < rows; ++r) out[mv_row(s, i, r)] = s->local[r] * mv_isd(s, i, r);
  }
  free(proj);
}
static int mv_xstar_t(const void* c, const double* xi, double* out) {
  const orc_mv* s = (const orc_mv*)c;
  const int64_t N0 = s->N0;
  for (int i = 0; i < s->G; ++i) {
    const int64_t rows = s->M0 + (s->roff[i + 1] - s->roff[i]);
    for (int64_t r = 0; r < rows; ++r) s->local[r] = xi[mv_row(s, i, r)] * mv_isd(s, i, r);
    gemv_t(rows, N0, s->Q + s->qoff[i], rows, s->local, out + (int64_t)i * N0);
    int st = tri_solve(N0, s->R + (int64_t)i * N0 * N0, out + (int64_t)i * N0, 0);
    if (st) return st;
  }
  return ORC_OK;
}
static int mv_xstar(const void* c, const double* v, double* out) {
  const orc_mv* s = (const orc_mv*)c;
  const int64_t N0 = s->N0;
  for (int64_t i = 0; i < s->m + s->k; ++i) out[i] = 0.0;
  for (int i = 0; i < s->G; ++i) {
    const int64_t rows = s->M0 + (s->roff[i + 1] - s->roff[i]);
    memcpy(s->tvec, v + (int64_t)i * N0, sizeof(double) * (size_t)N0);
    int st = tri_solve(N0, s->R + (int64_t)i * N0 * N0, s->tvec, 1);
    if (st) return st;
    gemv(rows, N0, s->Q + s->qoff[i], rows, s->tvec, s->local);
    for (int64_t r = 0; r < rows; ++r) out[mv_row(s, i, r)] = s->local[r] * mv_isd(s, i, r);
  }
  return ORC_OK;
}

/* X v with X = embed_mvrglm's dense matrix (dense_matrix.cpp:69-79): column i N0 + j holds Z0(:, j) on
 * equation i's rows and a 1 on the constraint row of (i, j) when j is restricted. */
static void mv_x(const void* c, const double* v, double* y) {
  const orc_mv* s = (const orc_mv*)c;
  for (int i = 0; i < s->G; ++i) gemv(s->M0, s->N0, s->Z0, s->M0, v + (int64_t)i * s->N0, y + (int64_t)i * s->M0);
  for (int i = 0; i < s->G; ++i)
    for (int64_t q = s->roff[i]; q < s->roff[i + 1]; ++q) {
      const double vj = v[(int64_t)i * s->N0 + s->ridx[q]];
      y[s->m + q] = (vj == 0.0) ? 0.0 : 0.0 + 1.0 * vj;
    }
}
/* X' w: per column, the sequential dot over every row (dense_matrix.cpp:81-91): the observation rows,
 * then the one constraint row */
static void mv_xt(const void* c, const double* w, double* out) {
  const orc_mv* s = (const orc_mv*)c;
  for (int i = 0; i < s->G; ++i) {
    double* oi = out + (int64_t)i * s->N0;
    gemv_t(s->M0, s->N0, s->Z0, s->M0, w + (int64_t)i * s->M0, oi);
    for (int64_t q = s->roff[i]; q < s->roff[i + 1]; ++q) oi[s->ridx[q]] += 1.0 * w[s->m + q];
  }
}
/* |X|_F in storage order (dense_matrix.cpp:93-97) */
static double mv_frob(const void* c) {
  const orc_mv* s = (const orc_mv*)c;
  double acc = 0.0;
  for (int i = 0; i < s->G; ++i) {
    int64_t q = s->roff[i];
    for (int64_t j = 0; j < s->N0; ++j) {
      for (int64_t r = 0; r < s->M0; ++r) acc += s->Z0[r + j * s->M0] * s->Z0[r + j * s->M0];
      if (q < s->roff[i + 1] && s->ridx[q] == j) { acc += 1.0 * 1.0; ++q; }
    }
  }
  return sqrt(acc);
}
/* Sigma = block_zero_padded(kronecker(Omega0, I_M0), k) (operators.cpp:51-57): the top is the dense
 * Kronecker matrix, whose row (a M0 + r) sums Omega0(a, b) x[b M0 + r] in ascending b -- the Kronecker
 * apply's order for a symmetric Omega0; the k constraint rows are zero. */
static void mv_sigma(const void* c, const double* x, double* out) {
  const orc_mv* s = (const orc_mv*)c;
  orc_kron_apply(s->G, s->M0, s->omega, x, out);
  for (int64_t q = 0; q < s->k; ++q) out[s->m + q] = 0.0;
}

int orc_pcg_aug_mvrglm(int G, int64_t M0, int64_t N0, const double* Z0, const double* Y, const double* omega,
                       const int64_t* roff, const int64_t* ridx, const double* z_scale, const double* c_scale,
                       const double* w1, const double* z1, const orc_config* cfg, const double* beta_true,
                       double* b_out, double* w_out, orc_trace_row* rows, int64_t rows_cap, orc_result* res,
                       int* bad_block) {
  orc_mv* s = NULL;
  int st = orc_mv_build(G, M0, N0, Z0, omega, roff, ridx, z_scale, c_scale, &s, bad_block);
  if (st) return st;
  const int64_t mt = s->m + s->k;
  double* y = (double*)calloc((size_t)mt, sizeof(double));
  if (!y) { orc_mv_free(s); return ORC_NO_MEMORY; }
  memcpy(y, Y, sizeof(double) * (size_t)s->m); /* y = [vec Y ; 0_k] (structured.cpp:89-90) */
  orc_model mo = {mt, s->n, s, mv_x, mv_xt, mv_frob, mv_sigma, mv_pi, mv_xstar_t, mv_xstar};
  st = run_aug(&mo, y, w1, z1, cfg, beta_true, b_out, w_out, rows, rows_cap, res);
  free(y);
  orc_mv_free(s);
  return st;
}

/* kind: 0 = apply_pi (m + k -> m + k), 1 = apply_xstar_t (-> G N0), 2 = apply_xstar (G N0 -> m + k);
 * 3 = Sigma apply, 4 = X apply (G N0 -> m + k), 5 = X' apply (m + k -> G N0) */
int orc_mvrglm_apply(int G, int64_t M0, int64_t N0, const double* Z0, const double* omega, const int64_t* roff,
                     const int64_t* ridx, const double* z_scale, const double* c_scale, int kind, const double* in,
                     double* out) {
  orc_mv* s = NULL;
  int bad = -1;
  int st = orc_mv_build(G, M0, N0, Z0, omega, roff, ridx, z_scale, c_scale, &s, &bad);
  if (st) return st;
  if (kind == 0) mv_pi(s, in, out);
  else if (kind == 1) st = mv_xstar_t(s, in, out);
  else if (kind == 2) st = mv_xstar(s, in, out);
  else if (kind == 3) mv_sigma(s, in, out);
  else if (kind == 4) mv_x(s, in, out);
  else mv_xt(s, in, out);
  orc_mv_free(s);
  return st;
}

double orc_mvrglm_norm_probe(int G, int64_t M0, int64_t N0, const double* Z0, const double* omega,
                             const int64_t* roff, const int64_t* ridx) {
  orc_mv* s = NULL;
  int bad = -1;
  if (orc_mv_build(G, M0, N0, Z0, omega, roff, ridx, NULL, NULL, &s, &bad)) return -1.0;
  orc_model mo = {s->m + s->k, s->n, s, mv_x, mv_xt, mv_frob, mv_sigma, mv_pi, mv_xstar_t, mv_xstar};
  const double r = model_norm_probe(&mo, 12);
  orc_mv_free(s);
  return r;
}

/* mv_reduce (structured.cpp:121-130): Z0 = Q0 R0; reduced Z0 = R0 (N0 x N0), reduced Y = Q0' Y via
 * DenseMatrix operator* (dense_matrix.cpp:125-139: out(:, j) += A(:, p) B(p, j), p ascending, skipping
 * B(p, j) == 0) with A = Q0' */
int orc_mv_reduce(int G, int64_t M0, int64_t N0, const double* Z0, const double* Y, double* r_out, double* qty_out) {
  double* q = (double*)malloc(sizeof(double) * (size_t)(M0 * N0));
  if (!q) return ORC_NO_MEMORY;
  int st = orc_qr_thin(M0, N0, Z0, M0, 1.0, q, M0, r_out);
  if (st) { free(q); return st; }
  for (int64_t k = 0; k < N0 * G; ++k) qty_out[k] = 0.0;
  for (int j = 0; j < G; ++j) {
    double* cj = qty_out + (int64_t)j * N0;
    for (int64_t p = 0; p < M0; ++p) {
      const double bpj = Y[p + (int64_t)j * M0];
      if (bpj == 0.0) continue;
      for (int64_t i = 0; i < N0; ++i) cj[i] += q[p + i * M0] * bpj; /* Q0'(i, p) = Q0(p, i) */
    }
  }
  free(q);
  return ORC_OK;
}

/* ------------------------------------------------------------------ PCG-NE on the SUR model
 * pcg_normal_equations(embed_sur(sur), nullptr, cfg, true_beta) (proj/src/pcg.cpp:364-511): CG on
 * X' Sigma^-1 X b = X' Sigma^-1 y with the identity preconditioner.  The reference factors the dense m x m
 * Sigma = Omega (x) I_M (cholesky, linalg.cpp:174-193); that factor is L (x) I_M with L = cholesky(Omega) by
 * the same loop (the off-pattern terms subtract exact zeros), and its chol_solve (linalg.cpp:195-210) is,
 * row by row of reshape(v, M, G), the G-dimensional forward / backward substitution with L, summed in the
 * same ascending order.  So the restatement never forms the m x m matrix. */
#define ORC_SINGULAR_COVARIANCE 5

static int chol_g(int G, const double* omega, double* L) {
  double max_diag = 0.0;
  for (int i = 0; i < G; ++i) max_diag = fmax(max_diag, fabs(omega[i + i * G]));
  const double floor_ = 64.0 * DBL_EPSILON * max_diag;
  for (int64_t k = 0; k < (int64_t)G * G; ++k) L[k] = 0.0;
  for (int j = 0; j < G; ++j) {
    double d = omega[j + j * G];
    for (int k = 0; k < j; ++k) d -= L[j + k * G] * L[j + k * G];
    if (d <= floor_) return ORC_SINGULAR_COVARIANCE;
    L[j + j * G] = sqrt(d);
    for (int i = j + 1; i < G; ++i) {
      double v = omega[i + j * G];
      for (int k = 0; k < j; ++k) v -= L[i + k * G] * L[j + k * G];
      L[i + j * G] = v / L[j + j * G];
    }
  }
  return ORC_OK;
}

/* x = (L L')^-1 x for Sigma = (L L') (x) I_M, in place; x is M x G column-major */
static void chol_solve_kron(int G, int64_t M, const double* L, double* x) {
  for (int64_t r = 0; r < M; ++r) {
    for (int i = 0; i < G; ++i) {
      double s = x[r + (int64_t)i * M];
      for (int j = 0; j < i; ++j) s -= L[i + j * G] * x[r + (int64_t)j * M];
      x[r + (int64_t)i * M] = s / L[i + i * G];
    }
    for (int i = G; i-- > 0;) {
      double s = x[r + (int64_t)i * M];
      for (int j = i + 1; j < G; ++j) s -= L[j + i * G] * x[r + (int64_t)j * M];
      x[r + (int64_t)i * M] = s / L[i + i * G];
    }
  }
}

int orc_pcg_ne_sur(int G, int64_t M, const int64_t* nb, const double* X, const double* Y, const double* omega,
                   const orc_config* cfg, const double* beta_true, double* b_out, double* w_out,
                   orc_trace_row* rows, int64_t rows_cap, orc_result* res) {
  const int64_t m = M * G, n = total_params(G, nb);
  double* L = (double*)malloc(sizeof(double) * (size_t)G * G);
  if (!L) return ORC_NO_MEMORY;
  int st = chol_g(G, omega, L);
  if (st) { free(L); return st; }
  const int64_t start = now_ns();
  const int64_t max_iter = cfg->max_iter ? cfg->max_iter : 2 * n;
  const int64_t stride = cfg->record_z_every ? cfg->record_z_every : 1;
  size_t mb = sizeof(double) * (size_t)m, nbytes = sizeof(double) * (size_t)n;
  double *tm = malloc(mb), *v = malloc(nbytes), *x = malloc(nbytes), *f = malloc(nbytes), *kf = malloc(nbytes),
         *p = malloc(nbytes), *gp = malloc(nbytes), *x_best = malloc(nbytes), *h = malloc(nbytes);
  if (!tm || !v || !x || !f || !kf || !p || !gp || !x_best || !h) { st = ORC_NO_MEMORY; goto done; }
  res->w1_projected = 0;
  res->breakdown_iteration = -1;
#define APPLY_G(in, out)                       \
  do {                                         \
    x_apply(G, M, nb, X, (in), tm);            \
    chol_solve_kron(G, M, L, tm);              \
    x_apply_t(G, M, nb, X, tm, (out));         \
  } while (0)
  /* crude norm probe for the breakdown scale (pcg.cpp:381-392) */
  double g_scale = 0.0;
  for (int64_t k = 0; k < n; ++k) v[k] = 1.0 / sqrt((double)n);
  for (int it = 0; it < 12; ++it) {
    APPLY_G(v, gp);
    memcpy(v, gp, nbytes);
    g_scale = vnorm2(n, v);
    if (g_scale == 0.0) break;
    for (int64_t k = 0; k < n; ++k) v[k] /= g_scale;
  }
  res->sigma_scale = g_scale;
  /* h = X' Sigma^-1 y; x = 0; f = -h; kf = f (no preconditioner) */
  memcpy(tm, Y, mb);
  chol_solve_kron(G, M, L, tm);
  x_apply_t(G, M, nb, X, tm, h);
  for (int64_t k = 0; k < n; ++k) { x[k] = 0.0; f[k] = -1.0 * h[k]; }
  memcpy(kf, f, nbytes);
  double c = vdot(n, f, kf);
  if (c < 0.0) c = 0.0;
  const double c1 = c, threshold = cfg->tol_rel * cfg->tol_rel * c1;
  memcpy(p, kf, nbytes);
  double k_gain = 0.0;
#define NE_FLOOR(fn2, kfn)                                                         \
  ((fn2) > 0.0 ? (k_gain = fmax(k_gain, (kfn) / sqrt(fn2))) : 0.0,                \
   16.0 * DBL_EPSILON * fmax(k_gain, 1e-3) * (fn2))
  (void)NE_FLOOR(vdot(n, f, f), vnorm2(n, kf));
  int64_t nrows = 0;
#define NE_ROW(iter_, cval_, sampled_)                                                          \
  do {                                                                                          \
    if (rows && nrows < rows_cap) {                                                             \
      orc_trace_row* row_ = &rows[nrows];                                                       \
      row_->iter = (iter_);                                                                     \
      row_->c = (cval_);                                                                        \
      row_->aug_residual_norm = vnorm2(n, f);                                                   \
      row_->dual_feas_norm = vnorm2(n, f);                                                      \
      if ((sampled_) && beta_true) {                                                            \
        double acc_ = 0.0;                                                                      \
        for (int64_t k_ = 0; k_ < n; ++k_) { const double d_ = x[k_] - beta_true[k_]; acc_ += d_ * d_; } \
        row_->rmse = sqrt(acc_ / (double)n);                                                    \
      } else {                                                                                  \
        row_->rmse = NAN;                                                                       \
      }                                                                                         \
      row_->elapsed_ns = now_ns() - start;                                                      \
    }                                                                                           \
    ++nrows;                                                                                    \
  } while (0)
  NE_ROW(0, c, 1);
  memcpy(x_best, x, nbytes);
  double c_best = c;
  int64_t best_iter = 0, stagnant = 0, done_it = 0;
  int term = T_MAXITER;
  if (c1 == 0.0) {
    term = T_CONVERGED;
  } else {
    for (int64_t i = 1; i <= max_iter; ++i) {
      APPLY_G(p, gp);
      const double d = vdot(n, p, gp);
      if (fabs(d) <= cfg->breakdown_tol * vdot(n, p, p) * fmax(g_scale, 1e-300)) {
        term = T_BREAKDOWN;
        res->breakdown_iteration = i;
        break;
      }
      const double lambda = c / d;
      for (int64_t k = 0; k < n; ++k) x[k] += -lambda * p[k];
      for (int64_t k = 0; k < n; ++k) f[k] += -lambda * gp[k];
      memcpy(kf, f, nbytes);
      double c_next = vdot(n, f, kf);
      done_it = i;
      const int sampled = (i % stride == 0) || c_next <= threshold || i == max_iter;
      NE_ROW(i, c_next, sampled);
      const double floor_c = NE_FLOOR(vdot(n, f, f), vnorm2(n, kf));
      const int exhausted = fabs(c_next) <= floor_c / 64.0 || (fabs(c_next) <= floor_c && c_next <= 1e-6 * c);
      if (c_next < 0.0 && fabs(c_next) > floor_c) {
        term = T_BREAKDOWN;
        res->breakdown_iteration = i;
        break;
      }
      if (c_next < 0.0) c_next = 0.0;
      if (c_next < c_best) {
        c_best = c_next;
        memcpy(x_best, x, nbytes);
        best_iter = i;
      }
      if (c_next <= threshold || exhausted) {
        term = T_CONVERGED;
        break;
      }
      if (fabs(c_next - c) <= 1e-15 * c) {
        if (++stagnant >= cfg->stagnation_window) {
          term = T_STAGNATION;
          break;
        }
      } else {
        stagnant = 0;
      }
      if (c_next > cfg->growth_tol * c_best && i - best_iter >= cfg->growth_window) {
        term = T_BREAKDOWN;
        res->breakdown_iteration = i;
        break;
      }
      const double mu = c_next / c;
      c = c_next;
      for (int64_t k = 0; k < n; ++k) p[k] = kf[k] + mu * p[k];
    }
  }
  {
    const int keep_last = term == T_CONVERGED;
    const double* b = keep_last ? x : x_best;
    memcpy(b_out, b, nbytes);
    if (w_out) { /* implied_w(b) = Sigma^-1 (y - X b) */
      x_apply(G, M, nb, X, b, tm);
      for (int64_t k = 0; k < m; ++k) w_out[k] = Y[k] - tm[k];
      chol_solve_kron(G, M, L, w_out);
    }
    res->iterations = done_it;
    res->termination = term;
    res->residual_seminorm = keep_last ? c : c_best;
    res->n_rows = nrows;
  }
#undef APPLY_G
#undef NE_FLOOR
#undef NE_ROW
done:
  free(L); free(tm); free(v); free(x); free(f); free(kf); free(p); free(gp); free(x_best); free(h);
  return st;
}
