// ne.cuh -- device-resident PCG-NE (pcg_normal_equations, /root/reference/proj/src/pcg.cpp:364-511) on the SUR model.
//
// CG on X' Sigma^-1 X b = X' Sigma^-1 y with the identity preconditioner.  Per iteration:
//   gp = X' chol_solve(L (x) I, X p)   -- k_xapply, k_chol_solve_kron, the X' column pass + k_reduce_t
//   k_ne_step                          -- d = p.gp, the breakdown test, x -= lambda p, f -= lambda gp, c = f.f,
//                                         the trace row, the floor / exhausted / negative-c / best / stagnation /
//                                         growth tests, mu, p = f + mu p (pcg.cpp:441-493), one CTA
// all on the device (the SolveState of the SUR solve carries the scalars), captured into CUDA graphs of `chunk`
// iterations like glsgpu_sur_solve; the host only polls `active` between graph launches.
//
// Sigma^-1 v is the reference's chol_solve (linalg.cpp:195-210) on the dense factor of Sigma = Omega (x) I_M, which
// is L (x) I_M with L = cholesky(Omega) (the off-pattern terms subtract exact zeros): per row of reshape(v, M, G),
// the G-dimensional forward then backward substitution in the reference's ascending / descending order, with
// separate multiply and subtract (-fmad=false) -- bitwise the reference's per-row arithmetic.
#pragma once

namespace glsgpu {

// x = (L L')^-1 x in place, rows [0, M) of the M x G column-major x (ld ldm); Lr = L row-major (row i of L
// contiguous, the forward loop), Lc = L column-major (column i contiguous, the backward loop).  Thread = row; the
// block's T rows x G columns stay in shared memory; L is read as warp-uniform broadcasts.
__global__ void k_chol_solve_kron(int G, int64_t ldm, int64_t M, const double* __restrict__ Lr,
                                  const double* __restrict__ Lc, double* __restrict__ x, const SolveState* st) {
  if (st && !st->active) return;
  extern __shared__ double tile[];  // [G][T]
  const int T = blockDim.x, t = threadIdx.x;
  for (int64_t r0 = (int64_t)blockIdx.x * T; r0 < M; r0 += (int64_t)gridDim.x * T) {
    const int64_t r = r0 + t;
    const bool in = r < M;
    if (in)
      for (int j = 0; j < G; ++j) tile[j * T + t] = x[r + (int64_t)j * ldm];
    if (in) {
      for (int i = 0; i < G; ++i) {
        const double* li = Lr + (int64_t)i * G;
        double s = tile[i * T + t];
        for (int j = 0; j < i; ++j) s -= li[j] * tile[j * T + t];
        tile[i * T + t] = s / li[i];
      }
      for (int i = G; i-- > 0;) {
        const double* ci = Lc + (int64_t)i * G;
        double s = tile[i * T + t];
        for (int j = i + 1; j < G; ++j) s -= ci[j] * tile[j * T + t];
        tile[i * T + t] = s / ci[i];
      }
      for (int j = 0; j < G; ++j) x[r + (int64_t)j * ldm] = tile[j * T + t];
    }
  }
}

constexpr int NE_NT = 1024;

// one CTA: sums of n-vector products in a fixed order (thread-strided partials, then the block tree)
template <int K>
__device__ __forceinline__ void ne_block_sum(double (&v)[K], double* red /* [32][K] */) {
  block_sum<K>(v, red);
  __syncthreads();
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) red[k] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = red[k];
  __syncthreads();
}

// crude norm probe (pcg.cpp:381-392): g_scale = |gp|; v = gp / g_scale (st->cont = 0 once g_scale == 0)
__global__ void __launch_bounds__(NE_NT) k_ne_probe(SolveState* st, const double* gp, double* v, int64_t n) {
  if (!st->cont) return;
  __shared__ double red[32 * 2];
  double a[1] = {0.0};
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) a[0] += gp[k] * gp[k];
  ne_block_sum<1>(a, red);
  const double gs = sqrt(a[0]);
  if (threadIdx.x == 0) st->sigma_scale = gs;
  if (gs == 0.0) {
    if (threadIdx.x == 0) st->cont = 0;
    return;
  }
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) v[k] = gp[k] / gs;
}

__device__ __forceinline__ void ne_row(SolveState* st, TraceRowD* rows, int64_t idx, int64_t iter, double c,
                                       double fnorm, double rmse) {
  if (idx < st->rows_cap) {
    TraceRowD& r = rows[idx];
    r.iter = iter;
    r.c = c;
    r.aug = fnorm;   // normal-equation residual (pcg.cpp:424-425)
    r.dual = fnorm;
    r.rmse = rmse;
    r.elapsed_ns = (int64_t)(globaltimer() - st->t0);
  }
}

// x = 0, f = -h, kf = f, c = max(f.f, 0), c1, threshold, p = kf, the k_gain of c_floor, trace row 0 (pcg.cpp:396-421)
__global__ void __launch_bounds__(NE_NT) k_ne_init(SolveState* st, const double* h, double* x, double* f, double* p,
                                                   double* xb, const double* beta, TraceRowD* rows, int64_t n) {
  __shared__ double red[32 * 3];
  double a[2] = {0.0, 0.0};
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
    const double fk = -1.0 * h[k];
    x[k] = 0.0;
    xb[k] = 0.0;
    f[k] = fk;
    p[k] = fk;
    a[0] += fk * fk;
    if (beta) a[1] += beta[k] * beta[k];  // rmse of x = 0
  }
  ne_block_sum<2>(a, red);
  if (threadIdx.x == 0) {
    const double ff = a[0];
    double c = ff;
    if (c < 0.0) c = 0.0;
    st->c = c;
    st->c1 = c;
    st->c_best = c;
    st->threshold = st->tol_rel * st->tol_rel * c;
    const double kfn = sqrt(ff);
    if (ff > 0.0) st->pi_gain = dmax_std(st->pi_gain, kfn / sqrt(ff));
    ne_row(st, rows, 0, 0, c, sqrt(ff), beta ? sqrt(a[1] / (double)n) : __longlong_as_double(0x7ff8000000000000LL));
    st->done = 0;
    st->i = 1;
    if (c == 0.0) {
      st->term = T_CONVERGED;
      st->active = 0;
    }
  }
}

// one CG step on the normal equations (pcg.cpp:441-493), gp = G p already formed
__global__ void __launch_bounds__(NE_NT) k_ne_step(SolveState* st, const double* gp, double* x, double* f, double* p,
                                                   double* xb, const double* beta, TraceRowD* rows, int64_t n) {
  if (!st->active) return;
  if (!st->have_beta) beta = nullptr;
  __shared__ double red[32 * 3];
  __shared__ int flag[2];
  const int64_t i = st->i;
  double a[2] = {0.0, 0.0};
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
    a[0] += p[k] * gp[k];
    a[1] += p[k] * p[k];
  }
  ne_block_sum<2>(a, red);
  const double d = a[0];
  if (fabs(d) <= st->breakdown_tol * a[1] * dmax_std(st->sigma_scale, 1e-300)) {
    if (threadIdx.x == 0) {
      st->term = T_BREAKDOWN;
      st->breakdown_iter = i;
      st->active = 0;
    }
    return;
  }
  const double c = st->c;
  const double lambda = c / d;
  double b3[3] = {0.0, 0.0, 0.0};
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
    const double xk = x[k] + -lambda * p[k];
    const double fk = f[k] + -lambda * gp[k];
    x[k] = xk;
    f[k] = fk;
    b3[0] += fk * fk;
    if (beta) {
      const double e = xk - beta[k];
      b3[1] += e * e;
    }
  }
  ne_block_sum<3>(b3, red);
  double c_next = b3[0];
  const double ff = b3[0], fnorm = sqrt(ff);
  if (threadIdx.x == 0) {
    st->done = i;
    const bool sampled = (i % st->stride == 0) || c_next <= st->threshold || i == st->max_iter;
    ne_row(st, rows, i, i, c_next, fnorm,
           (sampled && beta) ? sqrt(b3[1] / (double)n) : __longlong_as_double(0x7ff8000000000000LL));
    // c_floor(f.f, |kf|) (pcg.cpp:408-412)
    if (ff > 0.0) st->pi_gain = dmax_std(st->pi_gain, fnorm / sqrt(ff));
    const double floor_c = 16.0 * 2.220446049250313e-16 * dmax_std(st->pi_gain, 1e-3) * ff;
    const bool exhausted = fabs(c_next) <= floor_c / 64.0 || (fabs(c_next) <= floor_c && c_next <= 1e-6 * c);
    int stop = 0, improve = 0;
    if (c_next < 0.0 && fabs(c_next) > floor_c) {
      st->term = T_BREAKDOWN;
      st->breakdown_iter = i;
      stop = 1;
    } else {
      if (c_next < 0.0) c_next = 0.0;
      if (c_next < st->c_best) {
        st->c_best = c_next;
        st->best_iter = i;
        improve = 1;
      }
      if (c_next <= st->threshold || exhausted) {
        st->term = T_CONVERGED;
        stop = 1;
      } else {
        if (fabs(c_next - c) <= 1e-15 * c) {
          if (++st->stagnant >= st->stagnation_window) {
            st->term = T_STAGNATION;
            stop = 1;
          }
        } else {
          st->stagnant = 0;
        }
        if (!stop && c_next > st->growth_tol * st->c_best && i - st->best_iter >= st->growth_window) {
          st->term = T_BREAKDOWN;
          st->breakdown_iter = i;
          stop = 1;
        }
      }
    }
    if (stop) {
      st->active = 0;  // st->c stays the previous c: the reference breaks before c = c_next (pcg.cpp:472-497)
    } else {
      st->mu = c_next / c;
      st->c = c_next;
      st->i = i + 1;
      if (i + 1 > st->max_iter) {
        st->term = T_MAXITER;
        st->active = 0;
      }
    }
    flag[0] = stop;
    flag[1] = improve;
  }
  __syncthreads();
  const int stop = flag[0], improve = flag[1];
  if (improve)
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) xb[k] = x[k];
  if (stop) return;
  const double mu = st->mu;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) p[k] = f[k] + mu * p[k];
}

}  // namespace glsgpu
