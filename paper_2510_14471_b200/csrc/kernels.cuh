// kernels.cuh -- sm_100a device code of the B200-native SUR PCG-Aug solver.
//
// Compiled with -fmad=false: every a*b+c below is a separately rounded multiply and add, so the
// element-wise updates, the Kronecker apply (proj/src/operators.cpp:45-50 via dense_matrix.cpp:125-139),
// the row sums of X v / Q t (dense_matrix.cpp:69-79) and the triangular solves (linalg.cpp:119-145)
// round exactly as the reference's default x86-64 build does.  The long reductions over rows (dot
// products and Q'r) are fixed-shape trees: deterministic run to run, not the reference's sequential
// order (SURVEY.md s0.7 "parity envelope").
//
// Data layout in HBM: every M x G state vector and the concatenated Q / X are
// column-major with a padded leading dimension ldm = round_up(M, 32); padding rows are zero.
#pragma once
#include <type_traits>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace glsgpu {

constexpr unsigned FULL = 0xffffffffu;
constexpr int NT = 256;             // threads per CTA for the streaming passes
constexpr int GRID_CAP = 148 * 4;   // fixed (device-independent) grid of the grid-stride passes

// ------------------------------------------------------------------------------------------
// Geometry of one rank's row shard (device-visible, passed by value).
struct Geo {
  int G;
  int nch;          // row chunks per block for the column (Q'x) passes
  int64_t M;        // rows owned by this rank
  int64_t ldm;      // padded leading dimension of internal arrays
  int64_t n;        // total parameters
  int64_t CH;       // rows per chunk
  const int* nb;    // [G] widths
  const int64_t* p0;  // [G] first parameter of block b
  const int64_t* r0;  // [G] offset of R_b
  const double* wts;  // [G] w_b = 1/sqrt(block_scale_b): rows k < msig of block b
  const double* wtc;  // [G] weight of rows k >= msig (MVRGLM constraint rows, 1/sqrt(c_scale_b)); = wts for SUR
  int64_t msig;       // rows of every block under Sigma (SUR: ldm; MVRGLM: M0 -- the constraint rows below it
                      // have zero variance, Sigma = diag(Omega0 (x) I_M0, 0), operators.cpp:51-57)
};

// per-row weight of block b (Block::inv_sqrt_d, structured.cpp:287-292)
__device__ __forceinline__ double row_wgt(const Geo& g, double wz, double wc, int64_t k) { return k < g.msig ? wz : wc; }

// Solver state kept on the device; the scalar control of run_aug (proj/src/pcg.cpp:134-211)
// executes in k_scalar_a / k_scalar_c so no host round trip happens inside an iteration.
struct SolveState {
  double c, c1, threshold, c_best, pi_gain, lambda, mu, sigma_scale;
  double lam_prev;         // lambda of the w / sw update still pending (applied by the next pass A)
  double tol_rel, breakdown_tol, growth_tol;
  double d, uu, c_next, rr, prpr;
  int64_t i, max_iter, best_iter, stagnant, done, breakdown_iter, stride;
  int64_t stagnation_window, growth_window, diag_every;
  int64_t rows_cap;        // device trace capacity
  unsigned long long t0;   // %globaltimer at solve start
  int32_t active, term, cur, best, nxt, mu_pending, cont, diag_now, sampled, have_beta;
  // w_{i+1} = w_i - lambda_i u_i and sw_{i+1} = sw_i - lambda_i su_i (pcg.cpp:151-152) are deferred
  // to the next pass A (compute-bound, so their traffic is free there): upd_pending marks them
  int32_t upd_pending;
  // sw_mode 1 (k_kron_mma only): Sigma w is not carried by the recurrence sw -= lambda su (pcg.cpp:152) but
  // formed as Sigma w where it is read -- on trace-diagnostic rows and at the exit (b = X*'(y - Sigma w_sel))
  int32_t sw_direct;
};

struct TraceRowD {
  int64_t iter;
  double c, aug, dual, rmse;
  int64_t elapsed_ns;
};

enum { T_CONVERGED = 0, T_BREAKDOWN = 1, T_STAGNATION = 2, T_MAXITER = 3 };

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ double dmax_std(double a, double b) { return (a < b) ? b : a; }  // std::max

// Deterministic block reduction of K values (fixed shuffle tree, then warps in order).
template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double* red /* [NT/32][K] */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) v[k] += __shfl_xor_sync(FULL, v[k], s);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) red[warp * K + k] = v[k];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double a = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a += red[w * K + k];
      v[k] = a;
    }
  }
}

// Transpose-reduce NB per-lane accumulators across a warp: afterwards lane l holds the warp total
// of accumulator (l % NB).  Fixed butterfly: deterministic.
template <int NB>
__device__ __forceinline__ void warp_transpose_reduce(double (&acc)[NB]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 16; s >= NB; s >>= 1)
#pragma unroll
    for (int i = 0; i < NB; ++i) acc[i] += __shfl_xor_sync(FULL, acc[i], s);
#pragma unroll
  for (int s = NB / 2; s >= 1; s >>= 1) {
    const bool upper = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const double send = upper ? acc[i] : acc[i + s];
      const double keep = upper ? acc[i + s] : acc[i];
      acc[i] = keep + __shfl_xor_sync(FULL, send, s);
    }
  }
}

// ------------------------------------------------------------------------------------------
// Kronecker apply out = reshape(x, M, G) * Omega, i.e. (Omega (x) I_M) x   (operators.cpp:45-50).
// Tile: TR = 8 warps x RW rows, all G columns; lane owns columns c = lane + 32 q.  The p loop runs
// in ascending order from 0.0 with separate mul/add: bitwise the reference's operator* sum.
// Modes: in_mode 0: x = src; 1: x = src / (*div) (operator_norm_probe's v[i] /= nrm);
//        2: pass A: u_new = pr + mu*u when st->mu_pending (pcg.cpp:210) else u; writes u.
// Partials per CTA: [0] = sum x*out, [1] = sum x*x, [2] = sum out*out.
// column-block indices of the iteration vectors in the vector slab (glsgpu_sur::mvec)
enum { MV_W = 0, MV_SW = 3, MV_R = 6, MV_U = 7, MV_SU = 8, MV_PR = 9, MV_SPR = 10, MV_COUNT = 11 };

struct WBuf {
  double* w[3];
  double* sw[3];
};

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}

template <int CPL, int RW>
__global__ void __launch_bounds__(NT) k_kron(int G, int64_t ldm, int64_t ntiles, const double* __restrict__ omegaT,
                                             const double* src, const double* pr, const double* div, double* u_io,
                                             double* out, double* partials, int in_mode, const SolveState* st,
                                             WBuf wbuf, int64_t msig) {
  if (st && in_mode != 3 && !st->active) return;
  if (in_mode == 3) {  // Sigma w_cur into sw_cur on a diagnostics row (sw_mode 1; the last row comes after the stop)
    if (!st->diag_now) return;
    src = wbuf.w[st->cur];
    out = wbuf.sw[st->cur];
    partials = nullptr;
  }
  extern __shared__ double xs[];  // [G][TR]
  constexpr int TR = 8 * RW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double mu = 0.0, lp = 0.0;
  bool upd = false, wupd = false;
  double *wc = nullptr, *wn = nullptr, *swc = nullptr, *swn = nullptr;
  if (in_mode == 2) {
    upd = st->mu_pending != 0;
    mu = st->mu;
    wupd = st->upd_pending != 0;  // the deferred w / sw update of the previous iteration
    lp = st->lam_prev;
    wc = wbuf.w[st->cur];
    wn = wbuf.w[st->nxt];
    swc = wbuf.sw[st->cur];
    swn = wbuf.sw[st->nxt];
  }
  const double dv = (in_mode == 1) ? *div : 1.0;
  // G <= 128: Omega (G^2 doubles) lives in shared memory behind the tile, so the p loop's Omega reads are
  // shared-memory broadcasts instead of L1 / L2 round trips on the accumulation chain
  constexpr bool OMS = CPL <= 4;
  double* const oms = xs + G * TR;
  if (OMS) {
    for (int i = threadIdx.x; i < G * G; i += NT) oms[i] = omegaT[i];
    __syncthreads();
  }
  double p_xo = 0.0, p_xx = 0.0, p_oo = 0.0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t k0 = tile * TR;
    __syncthreads();
    if (in_mode == 2) {
      // batches of 4 elements per thread: every load of the batch is issued before any store, so the
      // deferred w / sw update (axpy(-lambda, u, w), axpy(-lambda, su, sw), pcg.cpp:151-152; su read
      // before Sigma u overwrites it) streams under the Kronecker math instead of serialising it
      const double* __restrict__ prr = pr;
      const double* __restrict__ wcr = wc;
      const double* __restrict__ swcr = swc;
      double* __restrict__ wnr = wn;
      double* __restrict__ swnr = swn;
      for (int idx0 = threadIdx.x; idx0 < G * TR; idx0 += 4 * NT) {
        double uo[4], pv[4], wv[4], swv[4], so[4];
        int64_t offs[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int idx = idx0 + e * NT;
          const int p = idx / TR, r = idx - p * TR;
          offs[e] = (int64_t)p * ldm + k0 + r;
          if (idx < G * TR) {
            uo[e] = u_io[offs[e]];
            pv[e] = upd ? prr[offs[e]] : 0.0;
            if (wupd) {
              wv[e] = wcr[offs[e]];
              swv[e] = swcr[offs[e]];
              so[e] = out[offs[e]];
            }
          }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int idx = idx0 + e * NT;
          if (idx < G * TR) {
            const int64_t off = offs[e];
            if (wupd) {
              wnr[off] = wv[e] + (-lp) * uo[e];
              swnr[off] = swv[e] + (-lp) * so[e];
            }
            double x = uo[e];
            if (upd) {
              x = pv[e] + mu * uo[e];
              u_io[off] = x;
            }
            const int p = idx / TR, r = idx - p * TR;
            xs[p * TR + r] = x;
          }
        }
      }
    } else {
      for (int idx = threadIdx.x; idx < G * TR; idx += NT) {
        const int p = idx / TR, r = idx - p * TR;
        const int64_t off = (int64_t)p * ldm + k0 + r;
        xs[p * TR + r] = (in_mode == 1) ? src[off] / dv : src[off];
      }
    }
    __syncthreads();
    double acc[RW][CPL];
#pragma unroll
    for (int i = 0; i < RW; ++i)
#pragma unroll
      for (int q = 0; q < CPL; ++q) acc[i][q] = 0.0;
    const int rbase = warp * RW;
    for (int p = 0; p < G; ++p) {
      double o[CPL];
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const int c = lane + 32 * q;
        o[q] = (c < G) ? (OMS ? oms[p * G + c] : __ldg(omegaT + (int64_t)p * G + c)) : 0.0;
      }
      double xr[RW];
#pragma unroll
      for (int i = 0; i < RW; ++i) xr[i] = xs[p * TR + rbase + i];
#pragma unroll
      for (int i = 0; i < RW; ++i)
#pragma unroll
        for (int q = 0; q < CPL; ++q) acc[i][q] = acc[i][q] + xr[i] * o[q];
    }
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const int c = lane + 32 * q;
      if (c < G) {
#pragma unroll
        for (int i = 0; i < RW; ++i) {
          // rows >= msig carry zero variance (MVRGLM constraint rows): Sigma x is 0 there
          const double o = (k0 + rbase + i < msig) ? acc[i][q] : 0.0;
          out[(int64_t)c * ldm + k0 + rbase + i] = o;
          const double x = xs[c * TR + rbase + i];
          p_xo += x * o;
          p_xx += x * x;
          p_oo += o * o;
        }
      }
    }
  }
  __shared__ double red[NT / 32 * 3];
  double v[3] = {p_xo, p_xx, p_oo};
  block_sum<3>(v, red);
  if (threadIdx.x == 0 && partials) {
    partials[blockIdx.x * 3 + 0] = v[0];
    partials[blockIdx.x * 3 + 1] = v[1];
    partials[blockIdx.x * 3 + 2] = v[2];
  }
}

// ------------------------------------------------------------------------------------------
// Tile constants of the FP64-bound pass A (k_kron_ws, 128 < G <= 256).
constexpr int KG_BM = 32;   // rows per tile
constexpr int KG_BK = 8;    // Omega rows per slab
constexpr int KG_LD = 256;  // Omega row stride in shared memory

// Sum K-wide partials of `count` CTAs in fixed order (one CTA); result to out[0..K).
template <int K>
__device__ __forceinline__ void reduce_partials(const double* partials, int count, double* out) {
  double v[K];
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x)
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] += partials[i * K + k];
  __shared__ double red[32 * K];
  block_sum<K>(v, red);
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) out[k] = v[k];
}

__global__ void k_reduce3(const double* partials, int count, double* out) { reduce_partials<3>(partials, count, out); }

// operator_norm_probe step (pcg.cpp:237-242): nrm = norm2(v); if 0 -> result 0 and stop.
__global__ void k_probe_step(const double* partials, int count, double* nrm, int* stop) {
  __shared__ double res[3];
  reduce_partials<3>(partials, count, res);
  if (threadIdx.x == 0) {
    if (*stop) return;
    const double s = sqrt(res[2]);
    *nrm = s;
    if (s == 0.0) *stop = 1;
  }
}

// ------------------------------------------------------------------------------------------
// Pass A scalar step (pcg.cpp:144-150): d = u.su, breakdown test, lambda = c/d.
__global__ void k_scalar_a(const double* partials, int count, SolveState* st) {
  if (!st->active) return;
  __shared__ double res[3];
  reduce_partials<3>(partials, count, res);
  if (threadIdx.x == 0) {
    if (st->upd_pending) {  // pass A just materialized w_i / sw_i into nxt
      st->cur = st->nxt;
      st->upd_pending = 0;
      int nx = 0;
      while (nx == st->cur || nx == st->best) ++nx;
      st->nxt = nx;
    }
    const double d = res[0], uu = res[1];
    st->d = d;
    st->uu = uu;
    if (fabs(d) <= st->breakdown_tol * uu * st->sigma_scale) {
      st->term = T_BREAKDOWN;
      st->breakdown_iter = st->i;
      st->active = 0;
      st->cont = 0;
      st->diag_now = 0;
      return;
    }
    st->lambda = st->c / d;
  }
}

// ------------------------------------------------------------------------------------------
// Column passes over (block, chunk) items: acc_j += A[k, j] * x_k for the rows of the chunk, then a
// deterministic transpose-reduce into tpart[(p0_b + j) * nch + ch].
//
// MODE_B   : pass B of an iteration (pcg.cpp:151-155): w -= lambda u, sw -= lambda su (into the
//            rotation buffer; now deferred to pass A), xv = X v (xv_mode X) or Q s / w_b (QR), r -= lambda(su + xv),
//            x = w_b * r  (gather of the following apply_pi / apply_xstar_t, structured.cpp:347-351).
// MODE_QT_R: x = w_b * r                    (apply_pi / apply_xstar_t of r)
// MODE_QT_D: x = w_b * (y - sw[sel])        (recover, pcg.cpp:96-98)
// MODE_QT_V: x = w_b * v                    (probe apply_xstar_t of a host vector)
// MODE_DIAG: A = X, x = w[cur] (X'w for dual_feas_norm, pcg.cpp:112); row part: resid = y - (sw + X est),
//            sum resid^2 -> rpart[b * nch + ch] (aug_residual_norm, pcg.cpp:108-111).
enum { MODE_B = 0, MODE_QT_R = 1, MODE_QT_D = 2, MODE_QT_V = 3, MODE_DIAG = 4 };

struct ColArgs {
  const double* A;      // matrix whose transpose is applied (Q, or X for MODE_DIAG)
  int64_t lda;
  const double* X;      // X for the X v row sums (xv_mode X) / diag
  int64_t ldx;
  const double* u;
  const double* su;
  double* wb[3];
  double* swb[3];
  double* r;
  const double* y;
  int64_t ldy;
  const double* vec;    // v (xv_mode X) / s (QR) for MODE_B; est for MODE_DIAG; input vector for QT_V
  const double* vin;    // MODE_QT_V input (m-vector, ld ldm)
  double* tpart;
  double* rpart;        // MODE_DIAG residual partials [G * nch]
  const int* blocks;    // block list of this launch
  int64_t avalid;       // rows of A that are valid (A = user X: M; internal Q: ldm)
  int xv_from_x;        // 1: xv = X v; 0: xv = Q s / w_b
  int sel_best;         // MODE_QT_D: use the selected final buffer (cur or best)
  int gate;             // 0: always run; 1: only while st->active; 2: only when st->diag_now
  int qdiag;            // MODE_DIAG with A = Q (xv_mode QR): X est = Q s / w, column partials Q' w
};

template <int MODE, bool FUSED>
__global__ void __launch_bounds__(NT) k_colpass(Geo g, ColArgs a, const SolveState* st) {
  if (a.gate == 1 && !st->active) return;
  if (a.gate == 2 && !st->diag_now) return;
  constexpr int NB = 32;
  extern __shared__ double xsm[];  // !FUSED: [CH] x values of the chunk
  __shared__ double red[NT / 32][NB];
  __shared__ double rred[NT / 32];
  __shared__ double svec_s[512];
  const int item = blockIdx.x;
  const int b = a.blocks[item / g.nch];
  const int ch = item % g.nch;
  const int nb = g.nb[b];
  const int64_t p0 = g.p0[b];
  const double wz = g.wts[b], wc = g.wtc[b];
  const int64_t k0 = (int64_t)ch * g.CH;
  const int64_t k1 = (k0 + g.CH < g.ldm) ? k0 + g.CH : g.ldm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  double lam = 0.0, lp = 0.0;  // lp: lambda of a pending w / sw update (applied on the fly)
  int cur = 0, selb = 0;
  if (MODE == MODE_B) lam = st->lambda;
  if (MODE == MODE_DIAG) cur = st->cur;
  if (MODE == MODE_QT_D) {
    if (a.sel_best) selb = (st->term == T_CONVERGED) ? st->cur : st->best;
    else selb = st->cur;
  }
  if ((MODE == MODE_DIAG || MODE == MODE_QT_D) && st && st->upd_pending) lp = st->lam_prev;
  if (MODE == MODE_B || MODE == MODE_DIAG) {
    for (int j = threadIdx.x; j < nb; j += NT) svec_s[j] = a.vec[p0 + j];
    __syncthreads();
  }
  const double* Ab = a.A + p0 * a.lda;
  const double* Xb = a.X ? a.X + p0 * a.ldx : nullptr;
  const int64_t vo = (int64_t)b * g.ldm;

  double acc[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) acc[j] = 0.0;
  double rsum = 0.0;

  // Row phase: compute x_k (and the side effects of the mode).
  for (int64_t k = k0 + threadIdx.x; k < k1; k += NT) {
    const int64_t off = vo + k;
    const double wgt = row_wgt(g, wz, wc, k);
    double x;
    double qv[NB];
    if (FUSED) {
#pragma unroll
      for (int j = 0; j < NB; ++j) qv[j] = (j < nb && k < a.avalid) ? Ab[(int64_t)j * a.lda + k] : 0.0;
    }
    if (MODE == MODE_B) {
      // (w / sw updates are deferred to the next pass A)
      const double suv = a.su[off], rv = a.r[off];
      double xv = 0.0;
      if (a.xv_from_x) {
        if (k < g.M)
          for (int j = 0; j < nb; ++j) xv = xv + Xb[(int64_t)j * a.ldx + k] * svec_s[j];
      } else {
        if (FUSED) {
#pragma unroll
          for (int j = 0; j < NB; ++j)
            if (j < nb) xv = xv + qv[j] * svec_s[j];
        } else {
          for (int j = 0; j < nb; ++j) xv = xv + Ab[(int64_t)j * a.lda + k] * svec_s[j];
        }
        xv = xv / wgt;
      }
      const double rn = rv - lam * (suv + xv);
      a.r[off] = rn;
      x = rn * wgt;
    } else if (MODE == MODE_QT_R) {
      x = a.r[off] * wgt;
    } else if (MODE == MODE_QT_D) {
      const double yv = (k < g.M) ? a.y[(int64_t)b * a.ldy + k] : 0.0;
      x = (yv - (a.swb[selb][off] + (-lp) * a.su[off])) * wgt;
    } else if (MODE == MODE_QT_V) {
      x = a.vin[off] * wgt;
    } else {  // MODE_DIAG
      double xe = 0.0;
      if (FUSED) {
#pragma unroll
        for (int j = 0; j < NB; ++j)
          if (j < nb) xe = xe + qv[j] * svec_s[j];
      } else {
        if (k < a.avalid)
          for (int j = 0; j < nb; ++j) xe = xe + Ab[(int64_t)j * a.lda + k] * svec_s[j];
      }
      if (a.qdiag) xe = xe / wgt;
      const double yv = (k < g.M) ? a.y[(int64_t)b * a.ldy + k] : 0.0;
      const double res = yv - ((a.swb[cur][off] + (-lp) * a.su[off]) + xe);
      if (k < g.M) rsum += res * res;
      x = a.wb[cur][off] + (-lp) * a.u[off];
    }
    if (FUSED) {
#pragma unroll
      for (int j = 0; j < NB; ++j) acc[j] += qv[j] * x;
    } else {
      xsm[k - k0] = x;
    }
  }

  if (MODE == MODE_DIAG) {
    double v1[1] = {rsum};
    block_sum<1>(v1, rred);
    if (threadIdx.x == 0) a.rpart[(int64_t)b * g.nch + ch] = v1[0];
  }

  auto flush = [&](int j0) {
    warp_transpose_reduce<NB>(acc);
    __syncthreads();
    red[warp][lane] = acc[0];
    __syncthreads();
    if (threadIdx.x < NB && j0 + (int)threadIdx.x < nb) {
      double s = 0.0;
      for (int w = 0; w < NT / 32; ++w) s += red[w][threadIdx.x];
      a.tpart[(p0 + j0 + threadIdx.x) * g.nch + ch] = s;
    }
  };

  if (FUSED) {
    flush(0);
  } else {
    __syncthreads();
    for (int j0 = 0; j0 < nb; j0 += NB) {
#pragma unroll
      for (int j = 0; j < NB; ++j) acc[j] = 0.0;
      for (int64_t k = k0 + threadIdx.x; k < k1; k += NT) {
        const double x = xsm[k - k0];
#pragma unroll
        for (int j = 0; j < NB; ++j)
          if (j0 + j < nb && k < a.avalid) acc[j] += Ab[(int64_t)(j0 + j) * a.lda + k] * x;
      }
      flush(j0);
    }
  }
}

// ------------------------------------------------------------------------------------------
// TMA-staged streaming pass (Blackwell bulk-copy engine).  A persistent grid walks (block, chunk)
// items in tiles of T rows; warp 0 issues one cp.async.bulk per column segment of the matrix tile(s)
// (Q and/or X: T contiguous doubles each, column-major) and per vector segment into an S-stage
// shared-memory ring, completion tracked by one mbarrier per stage (expect_tx).  Phase 1 (thread per
// row) does the row work; phase 2 (warp per column) the Q'x column partial sums.  The memory-level
// parallelism comes from the ring, not from registers.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// explicit global-space streaming stores (no generic-address path; evict-first: the data is next
// read by a later pass, long after this one has streamed the rest of the vectors through L2)
__device__ __forceinline__ void stg_cs(double* p, double v) {
  asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void stg_cs2(double* p, double a, double b) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(a), "d"(b) : "memory");
}
// 2-D tensor-map load of one box (coordinates: inner = row, outer = column)
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// ------------------------------------------------------------------------------------------
// Pass A, warp-specialised (128 < G <= 256, G % 8 == 0): the Kronecker apply Sigma u = U Omega
// (operators.cpp:45-50) as an FP64 register-blocked product over 32-row tiles, with
//   * 8 math warps: 8 rows x 4 columns per thread (4 row groups x 2 column halves), operands of step
//     p + 1 loaded while step p's separate multiplies / adds issue (bitwise the reference's order:
//     every output accumulated p-ascending from 0.0, no FMA contraction);
//   * 1 loader warp: Omega' in KW_OK-row slabs (KW_OK G contiguous doubles each), one cp.async.bulk per slab
//     into a KW_OS-stage ring (full: tx bytes; empty: one arrival per math warp);
//   * KW_EW element warps: build the NEXT tile's U while the math warps run the current one.  Per 8-column
//     chunk it loads the 32 x 8 boxes of u, pr, w, sw, su (one 2-D TMA each, through the tensor map of
//     the vector slab; KW_ES-stage ring), then per element: the deferred w / sw update
//     (pcg.cpp:151-152), u = pr + mu u (pcg.cpp:210), u.u.
// The math warps write Sigma u and the u . Sigma u partials.  No CTA-wide barrier inside the tile loop.
constexpr int KW_MATH = 8;                          // math warps
constexpr int KW_EW = 3;                            // element warps (columns ew, ew + 3, ew + 6 of each 8-column chunk)
constexpr int KW_NT = (KW_MATH + 1 + KW_EW) * 32;   // + loader warp
constexpr int KW_OK = 8;                            // Omega rows per slab
constexpr int KW_OS = 3;                            // Omega slab stages
constexpr int KW_ES = 4;                            // element chunk stages
constexpr int KW_XS = 34;                           // U tile row stride (doubles per p; +2 pad: 8-way instead of
                                                    // 32-way bank conflicts in the epilogue's per-column reads)
constexpr int KW_XT = KG_LD * KW_XS;                // U tile doubles
constexpr int KW_EC = 5 * KG_BK * KG_BM;            // element chunk doubles: 5 vectors x 8 columns x 32 rows
constexpr size_t kw_smem_bytes() { return (size_t)(2 * KW_XT + KW_OS * KW_OK * KG_LD + KW_ES * KW_EC) * sizeof(double); }

// ring position: slot and phase parity advanced together (no division in the loops)
struct RingPos {
  int slot = 0;
  uint32_t phase = 0;
  __device__ __forceinline__ void next(int stages) {
    if (++slot == stages) {
      slot = 0;
      phase ^= 1u;
    }
  }
};

template <bool FMA>
__global__ void __launch_bounds__(KW_NT, 1) k_kron_ws(const __grid_constant__ CUtensorMap vmap, int G, int64_t ldm,
                                                     int64_t ntiles, const double* __restrict__ omegaT,
                                                     double* __restrict__ u_io, double* __restrict__ out,
                                                     double* partials, const SolveState* st, WBuf wbuf,
                                                     int64_t msig) {
  if (!st->active) return;
  extern __shared__ __align__(128) double ksm[];
  __shared__ __align__(8) uint64_t om_full[KW_OS], om_empty[KW_OS], el_full[KW_ES], el_empty[KW_ES], xs_full[2],
      xs_empty[2];
  __shared__ double red[KW_NT / 32][2];
  double* const xsb = ksm;                                // [2][KG_LD][KW_XS]
  double* const omb = ksm + 2 * KW_XT;                    // [KW_OS][KW_OK][G]
  double* const elb = omb + KW_OS * KW_OK * KG_LD;        // [KW_ES][5][KG_BK][KG_BM]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nslab = G / KG_BK;   // element chunks per tile
  const int nslab_o = G / KW_OK;  // Omega slabs per tile
  const int64_t ntl = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;  // tiles of this CTA
  if (tid == 0) {
    for (int i = 0; i < KW_OS; ++i) {
      mbar_init(&om_full[i], 1);
      mbar_init(&om_empty[i], KW_MATH);
    }
    for (int i = 0; i < KW_ES; ++i) {
      mbar_init(&el_full[i], 1);
      mbar_init(&el_empty[i], KW_EW);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&xs_full[i], KW_EW * 32);
      mbar_init(&xs_empty[i], KW_MATH);
    }
    mbar_fence_init();
  }
  __syncthreads();
  double p_a = 0.0, p_b = 0.0;  // math warps: u . Sigma u; element warps: u . u
  if (warp == KW_MATH) {
    // ---------------- Omega loader
    if (lane == 0) {
      const uint32_t bytes = (uint32_t)(KW_OK * G * sizeof(double));
      RingPos w;
      int s = 0;
      for (int64_t g = 0; g < ntl * nslab_o; ++g) {
        if (g >= KW_OS) mbar_wait(&om_empty[w.slot], w.phase ^ 1u);
        mbar_expect_tx(&om_full[w.slot], bytes);
        tma_load_1d(omb + w.slot * KW_OK * KG_LD, omegaT + (int64_t)s * KW_OK * G, bytes, &om_full[w.slot]);
        w.next(KW_OS);
        if (++s == nslab_o) s = 0;
      }
    }
  } else if (warp > KW_MATH) {
    // ---------------- element warps: warp ew owns columns ew, ew + KW_EW, ... of every chunk; element
    // warp 0 lane 0 issues the chunk loads
    const int ew = warp - KW_MATH - 1;
    const bool upd = st->mu_pending != 0, wupd = st->upd_pending != 0;
    const double mu = st->mu, lp = st->lam_prev;
    // column-block bases of u, pr, w_cur, sw_cur, su in the vector slab
    const int cur = st->cur;
    const int bu = MV_U * G, bp = MV_PR * G, bw = (MV_W + cur) * G, bsw = (MV_SW + cur) * G, bsu = MV_SU * G;
    double* __restrict__ wn = wbuf.w[st->nxt];
    double* __restrict__ swn = wbuf.sw[st->nxt];
    const uint32_t chunk_bytes = (uint32_t)((1 + (upd ? 1 : 0) + (wupd ? 3 : 0)) * KG_BK * KG_BM * sizeof(double));
    const int64_t total = ntl * nslab;
    const bool issuer = (ew == 0 && lane == 0);
    RingPos ip;               // issue position
    int64_t e_issue = 0, it_tile = blockIdx.x;
    int it_c0 = 0;
    auto issue = [&]() {
      if (e_issue >= KW_ES) mbar_wait(&el_empty[ip.slot], ip.phase ^ 1u);
      double* E = elb + ip.slot * KW_EC;
      uint64_t* bar = &el_full[ip.slot];
      mbar_expect_tx(bar, chunk_bytes);
      const int row = (int)(it_tile * KG_BM);
      tma_load_2d(E, &vmap, row, bu + it_c0, bar);
      if (upd) tma_load_2d(E + 1 * KG_BK * KG_BM, &vmap, row, bp + it_c0, bar);
      if (wupd) {
        tma_load_2d(E + 2 * KG_BK * KG_BM, &vmap, row, bw + it_c0, bar);
        tma_load_2d(E + 3 * KG_BK * KG_BM, &vmap, row, bsw + it_c0, bar);
        tma_load_2d(E + 4 * KG_BK * KG_BM, &vmap, row, bsu + it_c0, bar);
      }
      ip.next(KW_ES);
      ++e_issue;
      it_c0 += KG_BK;
      if (it_c0 == G) {
        it_c0 = 0;
        it_tile += gridDim.x;
      }
    };
    if (issuer)
      while (e_issue < KW_ES - 1 && e_issue < total) issue();
    RingPos cp;               // consume position
    for (int64_t jl = 0; jl < ntl; ++jl) {
      const int b = (int)(jl & 1);
      if (jl >= 2) mbar_wait(&xs_empty[b], (uint32_t)(((jl >> 1) & 1) ^ 1));
      double* xs = xsb + b * KW_XT;
      const int64_t k0 = (blockIdx.x + jl * gridDim.x) * KG_BM;
      for (int k = 0; k < nslab; ++k) {
        if (issuer && e_issue < total) issue();
        mbar_wait(&el_full[cp.slot], cp.phase);
        const double* E = elb + cp.slot * KW_EC;
#pragma unroll
        for (int cc = ew; cc < KG_BK; cc += KW_EW) {
          const int c = k * KG_BK + cc;
          const int64_t off = (int64_t)c * ldm + k0 + lane;
          const double uo = E[(0 * KG_BK + cc) * KG_BM + lane];
          if (wupd) {
            stg_cs(wn + off, E[(2 * KG_BK + cc) * KG_BM + lane] + (-lp) * uo);
            stg_cs(swn + off, E[(3 * KG_BK + cc) * KG_BM + lane] + (-lp) * E[(4 * KG_BK + cc) * KG_BM + lane]);
          }
          double v = uo;
          if (upd) {
            v = E[(1 * KG_BK + cc) * KG_BM + lane] + mu * uo;
            stg_cs(u_io + off, v);
          }
          xs[c * KW_XS + lane] = v;
          p_b += v * v;
        }
        // this warp's reads of the slot are done: release it to the issuer (generic reads before the
        // next async-proxy write into it)
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&el_empty[cp.slot]);
        cp.next(KW_ES);
      }
      __syncwarp();
      mbar_arrive(&xs_full[b]);
    }
  } else {
    // ---------------- math warps
    const int rg = warp & 3, chf = warp >> 2;
    const int cb = 128 * chf + 2 * lane;  // columns cb, cb + 1, cb + 64, cb + 65
    RingPos rp;
    for (int64_t jl = 0; jl < ntl; ++jl) {
      const int b = (int)(jl & 1);
      mbar_wait(&xs_full[b], (uint32_t)((jl >> 1) & 1));
      const double* xs = xsb + b * KW_XT;
      const int64_t k0 = (blockIdx.x + jl * gridDim.x) * KG_BM;
      double acc[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][q] = 0.0;
      for (int s = 0; s < nslab_o; ++s) {
        mbar_wait(&om_full[rp.slot], rp.phase);
        const double* xp = xs + s * KW_OK * KW_XS + 8 * rg;
        const double* op = omb + rp.slot * KW_OK * KG_LD + cb;
        double2 xa[4], oa[2];
#pragma unroll
        for (int h = 0; h < 4; ++h) xa[h] = *reinterpret_cast<const double2*>(xp + 2 * h);
        oa[0] = *reinterpret_cast<const double2*>(op);
        oa[1] = *reinterpret_cast<const double2*>(op + 64);
#pragma unroll
        for (int pp = 0; pp < KW_OK; ++pp) {
          double2 xb[4], ob[2];
          if (pp + 1 < KW_OK) {
#pragma unroll
            for (int h = 0; h < 4; ++h) xb[h] = *reinterpret_cast<const double2*>(xp + (pp + 1) * KW_XS + 2 * h);
            ob[0] = *reinterpret_cast<const double2*>(op + (pp + 1) * G);
            ob[1] = *reinterpret_cast<const double2*>(op + (pp + 1) * G + 64);
          }
          const double xr[8] = {xa[0].x, xa[0].y, xa[1].x, xa[1].y, xa[2].x, xa[2].y, xa[3].x, xa[3].y};
          const double o[4] = {oa[0].x, oa[0].y, oa[1].x, oa[1].y};
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[i][q] = FMA ? __fma_rn(xr[i], o[q], acc[i][q]) : acc[i][q] + xr[i] * o[q];
          if (pp + 1 < KW_OK) {
#pragma unroll
            for (int h = 0; h < 4; ++h) xa[h] = xb[h];
            oa[0] = ob[0];
            oa[1] = ob[1];
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&om_empty[rp.slot]);
        rp.next(KW_OS);
      }
      // outputs (8 consecutive rows per column: 4 x 16-byte stores) + u . Sigma u partials
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = cb + 64 * (q >> 1) + (q & 1);
        if (c < G) {
          double* dst = out + (int64_t)c * ldm + k0 + 8 * rg;
          const double* xc = xs + c * KW_XS + 8 * rg;
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int64_t row = k0 + 8 * rg + 2 * h;  // rows >= msig: zero variance (MVRGLM constraint rows)
            const double o0 = row < msig ? acc[2 * h][q] : 0.0, o1 = row + 1 < msig ? acc[2 * h + 1][q] : 0.0;
            stg_cs2(dst + 2 * h, o0, o1);
            const double2 x2 = *reinterpret_cast<const double2*>(xc + 2 * h);
            p_a += x2.x * o0;
            p_a += x2.y * o1;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&xs_empty[b]);
    }
  }
  // (d, u.u) partials of this CTA, fixed order (pcg.cpp:144-145)
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    p_a += __shfl_xor_sync(FULL, p_a, o);
    p_b += __shfl_xor_sync(FULL, p_b, o);
  }
  if (lane == 0) {
    red[warp][0] = p_a;
    red[warp][1] = p_b;
  }
  __syncthreads();
  if (tid == 0) {
    double a = 0.0, bb = 0.0;
    for (int w = 0; w < KW_NT / 32; ++w) {
      a += red[w][0];
      bb += red[w][1];
    }
    partials[blockIdx.x * 3 + 0] = a;
    partials[blockIdx.x * 3 + 1] = bb;
    partials[blockIdx.x * 3 + 2] = 0.0;
  }
}

// ------------------------------------------------------------------------------------------
// Pass A on the FP64 tensor cores (128 < G <= 256, G % 8 == 0; kron_fma): the same work as k_kron_ws with
// the Kronecker product Sigma u = U Omega issued as DMMA (mma.sync m16n8k4 .f64).  A DMMA chains its four
// products k = 0..3 as fused multiply-adds in ascending k (checked bitwise on this GPU against a sequential
// fma chain, scripts/micro/dmma_layout.cu), so each output is the p-ascending FMA chain from 0.0 that
// k_kron_ws<true> computes, with one instruction per 256 FMAs instead of 32.
//   * 64-row tiles: every vector segment the element warps move is 512 contiguous bytes (32-row tiles, 256-byte
//     segments, measured 8.1 ms against 7.5 ms at c4).
//   * U is handed over in 8-column chunks through a ring (KM_UR slots), not as a double-buffered tile: the
//     math of Omega slab s needs exactly U columns [8 s, 8 s + 8).
//   * 8 math warps, warp w owns output columns [32 w, 32 w + 32) of the tile: 4 m16 x 4 n8 DMMA blocks,
//     64 accumulators per lane.  A (U) and B (Omega) fragments come from shared memory with strides of 68 / 260
//     doubles, which make both fragment loads bank-conflict free.  u . Sigma u reads the tile's u back from
//     global memory (L2) in the epilogue.
//   * 1 loader warp: lane 0 streams Omega' in 8-row slabs (one 2 KB bulk copy per row into the padded slab),
//     lane 1 issues the element stages (KM_ES in flight).
//   * KM_EW element warps: per chunk, 64 x 8 boxes of u, pr, w, sw, su (2-D TMA, KM_ES-stage ring), then per
//     element the deferred w / sw update (pcg.cpp:151-152), u = pr + mu u (pcg.cpp:210), u.u -- each as one fused
//     multiply-add (kron_fma), like d = u . Sigma u in the epilogue.  An FP64 instruction issued by these warps
//     stalls the SM's DMMA pipe (measured: one extra FP64 instruction per element costs about 1 ms of the pass at
//     c4), so the element work is kept to three per element.
constexpr int KM_BM = 64;                           // rows per tile
constexpr int KM_EW = 3;                            // element warps
constexpr int KM_NT = (KW_MATH + 1 + KM_EW) * 32;
constexpr int KM_OK = 8;                            // Omega rows per slab = U columns per chunk
constexpr int KM_OS = 4;                            // Omega slab stages
constexpr int KM_OLD = KG_LD + 4;                   // Omega slab row stride (doubles)
constexpr int KM_XS = KM_BM + 4;                    // U chunk stride per column (doubles)
constexpr int KM_UC = KM_OK * KM_XS;                // U chunk doubles
constexpr int KM_UR = 16;                           // U chunk slots
constexpr int KM_ES = 4;                            // element chunk stages
constexpr int KM_EC = 5 * KM_OK * KM_BM;            // element chunk doubles: 5 vectors x 8 columns x 64 rows
constexpr int KM_REG_SIDE = 88;                     // setmaxnreg: loader + element warpgroup
constexpr int KM_REG_MATH = 208;                   // the two math warpgroups: 168 + (168 - 72) / 2
static_assert(KM_EW == 3 && KW_MATH == 8, "setmaxnreg works on warpgroups of four warps");
constexpr size_t km_smem_bytes() {
  return (size_t)(KM_UR * KM_UC + KM_OS * KM_OK * KM_OLD + KM_ES * KM_EC) * sizeof(double);
}

__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a0), "d"(a1), "d"(b0));
}

template <bool APPLY>
__global__ void __launch_bounds__(KM_NT, 1) k_kron_mma(const __grid_constant__ CUtensorMap vmap64, int G, int64_t ldm,
                                                       int64_t ntiles, const double* __restrict__ omegaT,
                                                       double* __restrict__ u_io, double* __restrict__ out,
                                                       double* partials, const SolveState* st, WBuf wbuf, int64_t msig,
                                                       int plain) {
  // APPLY = false: pass A (plain ignored).  APPLY: out = Sigma x, no updates, no partials, for x = column block
  // `plain` of the vector slab, or (plain == -2) x = w_cur into sw_cur on a diagnostics row (sw_mode 1).
  if (!APPLY && !st->active) return;
  if (APPLY && plain == -2) {
    if (!st->diag_now) return;
    out = wbuf.sw[st->cur];
  }
  extern __shared__ __align__(128) double ksm[];
  __shared__ __align__(8) uint64_t om_full[KM_OS], om_empty[KM_OS], el_full[KM_ES], el_empty[KM_ES], uc_full[KM_UR],
      uc_empty[KM_UR];
  __shared__ double red[KM_NT / 32][2];
  double* const ucb = ksm;                                // [KM_UR][KM_OK][KM_XS]
  double* const omb = ksm + KM_UR * KM_UC;                // [KM_OS][KM_OK][KM_OLD]
  double* const elb = omb + KM_OS * KM_OK * KM_OLD;       // [KM_ES][5][KM_OK][KM_BM]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nchunk = G / KM_OK;   // chunks (= Omega slabs) per tile
  const int64_t ntl = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;  // tiles of this CTA
  if (tid == 0) {
    for (int i = 0; i < KM_OS; ++i) {
      mbar_init(&om_full[i], 1);
      mbar_init(&om_empty[i], KW_MATH);
    }
    for (int i = 0; i < KM_ES; ++i) {
      mbar_init(&el_full[i], 1);
      mbar_init(&el_empty[i], KM_EW);
    }
    for (int i = 0; i < KM_UR; ++i) {
      mbar_init(&uc_full[i], KM_EW);
      mbar_init(&uc_empty[i], KW_MATH);
    }
    mbar_fence_init();
  }
  __syncthreads();
  // register reallocation between the warpgroups (launch: 168 per thread): the loader / element warpgroup gives up
  // registers, the two math warpgroups take them -- the 128 accumulator registers no longer spill and the epilogue
  // can hold a row block's u values
  double p_a = 0.0, p_b = 0.0;  // math warps: u . Sigma u; element warps: u . u
  if (warp >= KW_MATH) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(KM_REG_SIDE));
  if (warp == KW_MATH) {
    // ---------------- Omega loader: slab s = rows [8 s, 8 s + 8) of Omega', one bulk copy per row
    if (lane == 0) {
      const uint32_t row_bytes = (uint32_t)(G * sizeof(double));
      RingPos w;
      int s = 0;
      for (int64_t q = 0; q < ntl * nchunk; ++q) {
        if (q >= KM_OS) mbar_wait(&om_empty[w.slot], w.phase ^ 1u);
        mbar_expect_tx(&om_full[w.slot], row_bytes * KM_OK);
        double* dst = omb + w.slot * KM_OK * KM_OLD;
        const double* src = omegaT + (int64_t)s * KM_OK * G;
#pragma unroll
        for (int r = 0; r < KM_OK; ++r) tma_load_1d(dst + r * KM_OLD, src + (int64_t)r * G, row_bytes, &om_full[w.slot]);
        w.next(KM_OS);
        if (++s == nchunk) s = 0;
      }
    } else if (lane == 1) {
      // ---------------- element stages: chunk q = 64 x 8 boxes of u (and pr, w, sw, su as needed), KM_ES in flight
      const bool upd = !APPLY && st->mu_pending != 0, wupd = !APPLY && st->upd_pending != 0;
      const int cur = st->cur;
      const int bu = !APPLY ? MV_U * G : (plain == -2 ? (MV_W + cur) * G : plain * G);
      const int bp = MV_PR * G, bw = (MV_W + cur) * G, bsw = (MV_SW + cur) * G, bsu = MV_SU * G;
      const bool swd = st->sw_direct != 0;
      const uint32_t chunk_bytes =
          (uint32_t)((1 + (upd ? 1 : 0) + (wupd ? (swd ? 1 : 3) : 0)) * KM_OK * KM_BM * sizeof(double));
      RingPos ip;
      int64_t it_tile = blockIdx.x;
      int it_c0 = 0;
      for (int64_t q = 0; q < ntl * nchunk; ++q) {
        if (q >= KM_ES) mbar_wait(&el_empty[ip.slot], ip.phase ^ 1u);
        double* E = elb + ip.slot * KM_EC;
        uint64_t* bar = &el_full[ip.slot];
        mbar_expect_tx(bar, chunk_bytes);
        const int row = (int)(it_tile * KM_BM);
        tma_load_2d(E, &vmap64, row, bu + it_c0, bar);
        if (upd) tma_load_2d(E + 1 * KM_OK * KM_BM, &vmap64, row, bp + it_c0, bar);
        if (wupd) {
          tma_load_2d(E + 2 * KM_OK * KM_BM, &vmap64, row, bw + it_c0, bar);
          if (!swd) {
            tma_load_2d(E + 3 * KM_OK * KM_BM, &vmap64, row, bsw + it_c0, bar);
            tma_load_2d(E + 4 * KM_OK * KM_BM, &vmap64, row, bsu + it_c0, bar);
          }
        }
        ip.next(KM_ES);
        it_c0 += KM_OK;
        if (it_c0 == G) {
          it_c0 = 0;
          it_tile += gridDim.x;
        }
      }
    }
  } else if (warp > KW_MATH) {
    // ---------------- element warps: element i = (column i / 64, row i % 64) of a chunk, i = etid + 32 KM_EW e
    const int ew = warp - KW_MATH - 1;
    const int etid = ew * 32 + lane;
    const bool upd = !APPLY && st->mu_pending != 0, wupd = !APPLY && st->upd_pending != 0;
    const double mu = st->mu, lp = st->lam_prev;
    double* __restrict__ wn = wbuf.w[st->nxt];
    double* __restrict__ swn = wbuf.sw[st->nxt];
    const bool swd = st->sw_direct != 0;  // no sw recurrence: w alone is updated
    const bool fast = upd && wupd && swd;
    RingPos cp, up;
    constexpr int NE = (KM_OK * KM_BM + 32 * KM_EW - 1) / (32 * KM_EW);  // elements per thread per chunk
    for (int64_t jl = 0; jl < ntl; ++jl) {
      const int64_t k0 = (blockIdx.x + jl * gridDim.x) * KM_BM;
      for (int k = 0; k < nchunk; ++k) {
        mbar_wait(&el_full[cp.slot], cp.phase);
        if (jl * nchunk + k >= KM_UR) mbar_wait(&uc_empty[up.slot], up.phase ^ 1u);
        const double* E = elb + cp.slot * KM_EC;
        double* U = ucb + up.slot * KM_UC;
        if (fast && k0 + KM_BM <= ldm) {
          // the iteration's common case (u = pr + mu u, w -= lambda u, no sw recurrence, tile inside the matrix) as
          // straight-line code: every operand load first, then the fused multiply-adds back to back, then the stores
          // (u . u is summed by the math warps' epilogue from the u values it reads anyway)
          double uo[NE], pv[NE], wv[NE];
#pragma unroll
          for (int e = 0; e < NE; ++e) {
            const int i = etid + 32 * KM_EW * e;
            if (e == NE - 1 && (KM_OK * KM_BM) % (32 * KM_EW) != 0 && i >= KM_OK * KM_BM) break;
            uo[e] = E[i];
            pv[e] = E[KM_OK * KM_BM + i];
            wv[e] = E[2 * KM_OK * KM_BM + i];
          }
#pragma unroll
          for (int e = 0; e < NE; ++e) {
            const int i = etid + 32 * KM_EW * e;
            if (e == NE - 1 && (KM_OK * KM_BM) % (32 * KM_EW) != 0 && i >= KM_OK * KM_BM) break;
            wv[e] = __fma_rn(-lp, uo[e], wv[e]);
            pv[e] = __fma_rn(mu, uo[e], pv[e]);
          }
#pragma unroll
          for (int e = 0; e < NE; ++e) {
            const int i = etid + 32 * KM_EW * e;
            if (e == NE - 1 && (KM_OK * KM_BM) % (32 * KM_EW) != 0 && i >= KM_OK * KM_BM) break;
            const int cc = i / KM_BM, rr = i % KM_BM;
            const int64_t off = (int64_t)(k * KM_OK + cc) * ldm + k0 + rr;
            stg_cs(wn + off, wv[e]);
            u_io[off] = pv[e];  // read back by the math warps' epilogue (L2)
            U[cc * KM_XS + rr] = pv[e];
          }
        } else {
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          const int i = etid + 32 * KM_EW * e;
          if ((KM_OK * KM_BM) % (32 * KM_EW) != 0 && i >= KM_OK * KM_BM) break;
          const int cc = i / KM_BM, rr = i % KM_BM;
          const int c = k * KM_OK + cc;
          const int64_t grow = k0 + rr;
          const int64_t off = (int64_t)c * ldm + grow;
          const bool in = grow < ldm;
          const double uo = E[(0 * KM_OK + cc) * KM_BM + rr];
          if (wupd && in) {
            stg_cs(wn + off, __fma_rn(-lp, uo, E[(2 * KM_OK + cc) * KM_BM + rr]));
            if (!swd) stg_cs(swn + off, __fma_rn(-lp, E[(4 * KM_OK + cc) * KM_BM + rr], E[(3 * KM_OK + cc) * KM_BM + rr]));
          }
          double v = uo;
          if (upd) {
            v = __fma_rn(mu, uo, E[(1 * KM_OK + cc) * KM_BM + rr]);
            if (in) u_io[off] = v;  // read back by the math warps' epilogue (L2)
          }
          U[cc * KM_XS + rr] = v;
          p_b = __fma_rn(v, v, p_b);
        }
        }
        // this warp's reads of the element slot are done; its U chunk writes are published to the math warps (both by
        // the mbarrier arrivals' release; no proxy fence: it compiles to a MEMBAR that also waits for this chunk's
        // global stores, and a generic read followed by the next bulk copy into the slot is ordered by the barrier)
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&el_empty[cp.slot]);
          mbar_arrive(&uc_full[up.slot]);
        }
        cp.next(KM_ES);
        up.next(KM_UR);
      }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(KM_REG_MATH));
    // ---------------- math warps: DMMA m16n8k4, warp owns columns [32 warp, 32 warp + 32) of every tile
    const int g = lane >> 2, t = lane & 3;
    const int n0 = 32 * warp;
    // (the same condition as the element warps' `fast`)
    const bool uu_math = !APPLY && st->mu_pending != 0 && st->upd_pending != 0 && st->sw_direct != 0;
    RingPos rp, up;
    for (int64_t jl = 0; jl < ntl; ++jl) {
      const int64_t k0 = (blockIdx.x + jl * gridDim.x) * KM_BM;
      double acc[4][4][4];  // [m16 tile][n8 tile][fragment]
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[mi][ni][q] = 0.0;
      for (int s = 0; s < nchunk; ++s) {
        mbar_wait(&uc_full[up.slot], up.phase);
        mbar_wait(&om_full[rp.slot], rp.phase);
        const double* om = omb + rp.slot * KM_OK * KM_OLD + n0 + g;
        const double* U = ucb + up.slot * KM_UC + t * KM_XS + g;
#pragma unroll
        for (int kk = 0; kk < KM_OK / 4; ++kk) {
          const double* ob = om + (kk * 4 + t) * KM_OLD;
          const double b0 = ob[0], b1 = ob[8], b2 = ob[16], b3 = ob[24];
          const double* ua = U + kk * 4 * KM_XS;
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) {
            const double a0 = ua[16 * mi], a1 = ua[16 * mi + 8];
            dmma_16x8x4(acc[mi][0], a0, a1, b0);
            dmma_16x8x4(acc[mi][1], a0, a1, b1);
            dmma_16x8x4(acc[mi][2], a0, a1, b2);
            dmma_16x8x4(acc[mi][3], a0, a1, b3);
          }
        }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&om_empty[rp.slot]);
          mbar_arrive(&uc_empty[up.slot]);
        }
        rp.next(KM_OS);
        up.next(KM_UR);
      }
      // epilogue: acc[mi][ni] = rows 16 mi + (g, g + 8) x columns n0 + 8 ni + 2 t (+1); rows >= msig carry
      // zero variance; u . Sigma u with the tile's u from global memory (L2).  The registers setmaxnreg moved to
      // the math warps hold one m16 row block's 16 u values at a time: one L2 round trip per row block instead of
      // one per small group of loads behind the stores.
      const bool tile_in = k0 + KM_BM <= ldm && n0 + 32 <= G;
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        double uv[4][4];
        if (!APPLY) {
#pragma unroll
          for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int c = n0 + 8 * ni + 2 * t + (q & 1);
              const int64_t grow = k0 + 16 * mi + g + 8 * (q >> 1);
              uv[ni][q] = (tile_in || (c < G && grow < ldm)) ? u_io[(int64_t)c * ldm + grow] : 0.0;
            }
        }
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int c = n0 + 8 * ni + 2 * t + (q & 1);
            const int64_t grow = k0 + 16 * mi + g + 8 * (q >> 1);
            if (tile_in || (c < G && grow < ldm)) {
              const double o = grow < msig ? acc[mi][ni][q] : 0.0;
              stg_cs(out + (int64_t)c * ldm + grow, o);
              if (!APPLY) p_a = __fma_rn(uv[ni][q], o, p_a);
            }
          }
        if (!APPLY && uu_math && k0 + KM_BM <= ldm) {  // u . u of the tiles the element warps' fast path handled
#pragma unroll
          for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int q = 0; q < 4; ++q) p_b = __fma_rn(uv[ni][q], uv[ni][q], p_b);
        }
      }
    }
  }
  // (d, u.u) partials of this CTA, fixed order (pcg.cpp:144-145)
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    p_a += __shfl_xor_sync(FULL, p_a, o);
    p_b += __shfl_xor_sync(FULL, p_b, o);
  }
  if (lane == 0) {
    red[warp][0] = p_a;
    red[warp][1] = p_b;
  }
  __syncthreads();
  if (tid == 0 && !APPLY) {
    double a = 0.0, bb = 0.0;
    for (int w = 0; w < KM_NT / 32; ++w) {
      a += red[w][0];
      bb += red[w][1];
    }
    partials[blockIdx.x * 3 + 0] = a;
    partials[blockIdx.x * 3 + 1] = bb;
    partials[blockIdx.x * 3 + 2] = 0.0;
  }
}

// ------------------------------------------------------------------------------------------
// Pass A on the FP64 tensor cores, second form (round 2; the default): the math warps build their own A operands.
// k_kron_mma's element warps produced the U tile (u = pr + mu u) for the math warps through a shared-memory ring, so
// the DMMA stream waited on three warps whose every DFMA queues behind the math warps' DMMA bursts (ncu: the math
// warps 23% on the ring's full barriers, the element warps 27% on their loads and 17% on the first DFMA of a chunk).
// Here one ring of KM2 stages carries, per 8-column chunk, the Omega slab and the raw chunk columns of u_old, pr, w
// (and sw, su for the recurrence mode), every column one 512-byte bulk copy into a padded (conflict-free) layout:
//   * the 8 math warps read u_old and pr as fragments and form a = fma(mu, u_old, pr) inline (bitwise the element
//     warps' value; 16 DFMAs per 32 DMMAs per warp, issued by the warps that own the FP64 pipe);
//   * the 3 side warps only write: u (read back by the epilogue's u . Sigma u, after a per-tile barrier), the
//     deferred w (and sw) update, and u . u where the epilogue does not take it; they are off the DMMA stream's
//     critical path -- a stage is recycled when the math warps AND the side warps have released it;
//   * the loader warp: lanes 0-7 the Omega rows, lanes 8.. one chunk column each.
constexpr int KM2_MAXS = 12;                        // ring stages (barrier arrays)
constexpr int KM2_OM = KM_OK * KM_OLD;              // Omega slab doubles per stage
constexpr int KM2_VC = KM_OK * KM_XS;               // one vector's chunk, padded: [8 columns][68]
constexpr size_t km2_stage_bytes(int nv) { return (size_t)(KM2_OM + nv * KM2_VC) * sizeof(double); }

template <bool APPLY, int MW>
__global__ void __launch_bounds__((MW + 1 + KM_EW) * 32, 1) k_kron_mma2(const double* __restrict__ slab, int G, int64_t ldm,
                                                        int64_t ntiles, const double* __restrict__ omegaT,
                                                        double* __restrict__ u_io, double* __restrict__ out,
                                                        double* partials, const SolveState* st, WBuf wbuf,
                                                        int64_t msig, int plain, int nstage, int nv) {
  // APPLY = false: pass A (plain ignored).  APPLY: out = Sigma x, no updates, no partials, for x = column block
  // `plain` of the vector slab, or (plain == -2) x = w_cur into sw_cur on a diagnostics row (sw_mode 1).
  if (!APPLY && !st->active) return;
  if (APPLY && plain == -2) {
    if (!st->diag_now) return;
    out = wbuf.sw[st->cur];
  }
  // MW math warps (8: 32 columns each, 128 accumulator registers; 16: 16 columns each, 64 accumulator registers and
  // four math warps per scheduler to cover one another's DMMA issue gaps), one loader warp, KM_EW side warps
  constexpr int NTH = (MW + 1 + KM_EW) * 32;
  constexpr int NI = 32 / MW;                      // n8 column blocks per math warp
  // setmaxnreg.inc only draws on what setmaxnreg.dec released: (launch - side) * 128 >= (math - launch) * 32 MW
  constexpr int REG_LAUNCH = MW == 8 ? 168 : 96;
  constexpr int REG_SIDE = MW == 8 ? KM_REG_SIDE : 56, REG_MATH = MW == 8 ? KM_REG_MATH : 104;
  static_assert((REG_LAUNCH - REG_SIDE) * 128 >= (REG_MATH - REG_LAUNCH) * 32 * MW, "register pool");
  static_assert(MW == 8 || MW == 16, "math warp layouts");
  extern __shared__ __align__(128) double ksm[];
  __shared__ __align__(8) uint64_t full[KM2_MAXS], empty[KM2_MAXS], tile_done;
  __shared__ double red[NTH / 32][2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nchunk = G / KM_OK;   // chunks (= Omega slabs) per tile
  const int64_t ntl = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;  // tiles of this CTA
  const int sstride = KM2_OM + nv * KM2_VC;
  const bool upd = !APPLY && st->mu_pending != 0, wupd = !APPLY && st->upd_pending != 0;
  const bool swd = st->sw_direct != 0;  // no sw recurrence: w alone is updated
  const bool fast = upd && wupd;  // the iteration's common case: u . u moves to the math epilogue
  for (int i = tid; i < nstage * sstride; i += NTH) ksm[i] = 0.0;  // rows past a short last tile stay 0
  if (tid == 0) {
    for (int i = 0; i < nstage; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], MW + KM_EW);
    }
    mbar_init(&tile_done, KM_EW);
    mbar_fence_init();
  }
  fence_proxy_async_smem();
  __syncthreads();
  double p_a = 0.0, p_b = 0.0;  // u . Sigma u (math warps); u . u (math warps' epilogue, or the side warps)
  if (warp >= MW) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(REG_SIDE));
    if (warp == MW) {
      // ---------------- loader: per chunk, 8 Omega rows (lanes 0-7) and the chunk columns (lane 8 + 8 v + column)
      const int cur = st->cur;
      const int64_t mv = ldm * G;
      // stage vector v: 0 = u (or the plain vector), 1 = pr, 2 = w_cur, 3 = sw_cur, 4 = su; lanes 8..31 take
      // (vector, column) pairs idx = lane - 8 + 24 j
      auto v_on = [&](int v) { return v == 0 || (v == 1 && upd) || (v == 2 && wupd) || (v >= 3 && wupd && !swd); };
      auto v_src = [&](int v) {
        const int blk = v == 0 ? (!APPLY ? MV_U : (plain == -2 ? MV_W + cur : plain))
                        : v == 1 ? MV_PR : v == 2 ? MV_W + cur : v == 3 ? MV_SW + cur : MV_SU;
        return slab + (int64_t)blk * mv;
      };
      const int nvec_on = 1 + (upd ? 1 : 0) + (wupd ? (swd ? 1 : 3) : 0);
      const uint32_t om_bytes = (uint32_t)(G * sizeof(double)) * KM_OK;
      RingPos w;
      int64_t tile = blockIdx.x;
      int c0 = 0;
      for (int64_t q = 0; q < ntl * nchunk; ++q) {
        if (q >= nstage) mbar_wait(&empty[w.slot], w.phase ^ 1u);
        double* S = ksm + w.slot * sstride;
        const int64_t k0 = tile * KM_BM;
        const uint32_t col_bytes = (uint32_t)(min((int64_t)KM_BM, ldm - k0) * sizeof(double));
        if (lane == 0) mbar_expect_tx(&full[w.slot], om_bytes + (uint32_t)nvec_on * KM_OK * col_bytes);
        __syncwarp();
        if (lane < 8)
          tma_load_1d(S + lane * KM_OLD, omegaT + (int64_t)(c0 + lane) * G, (uint32_t)(G * sizeof(double)), &full[w.slot]);
        else
          for (int idx = lane - 8; idx < nv * KM_OK; idx += 24) {
            const int v = idx >> 3, lc = idx & 7;
            if (v_on(v))
              tma_load_1d(S + KM2_OM + v * KM2_VC + lc * KM_XS, v_src(v) + (int64_t)(c0 + lc) * ldm + k0, col_bytes,
                          &full[w.slot]);
          }
        w.next(nstage);
        c0 += KM_OK;
        if (c0 == G) {
          c0 = 0;
          tile += gridDim.x;
        }
      }
    } else {
      // ---------------- side warps: element i = (column i / 64, row i % 64) of a chunk, i = etid + 32 KM_EW e
      const int ew = warp - MW - 1;
      const int etid = ew * 32 + lane;
      const double mu = st->mu, lp = st->lam_prev;
      double* __restrict__ wn = wbuf.w[st->nxt];
      double* __restrict__ swn = wbuf.sw[st->nxt];
      RingPos cp;
      constexpr int NE = (KM_OK * KM_BM + 32 * KM_EW - 1) / (32 * KM_EW);  // elements per thread per chunk
      for (int64_t jl = 0; jl < ntl; ++jl) {
        const int64_t k0 = (blockIdx.x + jl * gridDim.x) * KM_BM;
        const bool tile_in = k0 + KM_BM <= ldm;
        for (int k = 0; k < nchunk; ++k) {
          mbar_wait(&full[cp.slot], cp.phase);
          const double* E = ksm + cp.slot * sstride + KM2_OM;
          if (fast && tile_in) {
            double uo[NE], pv[NE], wv[NE];
#pragma unroll
            for (int e = 0; e < NE; ++e) {
              const int i = etid + 32 * KM_EW * e;
              if (e == NE - 1 && (KM_OK * KM_BM) % (32 * KM_EW) != 0 && i >= KM_OK * KM_BM) break;
              const int o = (i / KM_BM) * KM_XS + i % KM_BM;
              uo[e] = E[o];
              pv[e] = E[KM2_VC + o];
              wv[e] = E[2 * KM2_VC + o];
            }
#pragma unroll
            for (int e = 0; e < NE; ++e) {
              const int i = etid + 32 * KM_EW * e;
              if (e == NE - 1 && (KM_OK * KM_BM) % (32 * KM_EW) != 0 && i >= KM_OK * KM_BM) break;
              wv[e] = __fma_rn(-lp, uo[e], wv[e]);
              pv[e] = __fma_rn(mu, uo[e], pv[e]);
            }
#pragma unroll
            for (int e = 0; e < NE; ++e) {
              const int i = etid + 32 * KM_EW * e;
              if (e == NE - 1 && (KM_OK * KM_BM) % (32 * KM_EW) != 0 && i >= KM_OK * KM_BM) break;
              const int64_t off = (int64_t)(k * KM_OK + i / KM_BM) * ldm + k0 + i % KM_BM;
              stg_cs(wn + off, wv[e]);
              u_io[off] = pv[e];  // read back by the math warps' epilogue (L2)
            }
            if (!swd) {  // Sigma w carried by the reference's recurrence (pcg.cpp:152): sw -= lambda su
#pragma unroll
              for (int e = 0; e < NE; ++e) {
                const int i = etid + 32 * KM_EW * e;
                if (e == NE - 1 && (KM_OK * KM_BM) % (32 * KM_EW) != 0 && i >= KM_OK * KM_BM) break;
                const int o = (i / KM_BM) * KM_XS + i % KM_BM;
                wv[e] = __fma_rn(-lp, E[4 * KM2_VC + o], E[3 * KM2_VC + o]);
              }
#pragma unroll
              for (int e = 0; e < NE; ++e) {
                const int i = etid + 32 * KM_EW * e;
                if (e == NE - 1 && (KM_OK * KM_BM) % (32 * KM_EW) != 0 && i >= KM_OK * KM_BM) break;
                stg_cs(swn + (int64_t)(k * KM_OK + i / KM_BM) * ldm + k0 + i % KM_BM, wv[e]);
              }
            }
          } else if (!APPLY) {
#pragma unroll
            for (int e = 0; e < NE; ++e) {
              const int i = etid + 32 * KM_EW * e;
              if ((KM_OK * KM_BM) % (32 * KM_EW) != 0 && i >= KM_OK * KM_BM) break;
              const int cc = i / KM_BM, rr = i % KM_BM;
              const int64_t grow = k0 + rr;
              const int64_t off = (int64_t)(k * KM_OK + cc) * ldm + grow;
              const bool in = grow < ldm;
              const int o = cc * KM_XS + rr;
              const double uo = in ? E[o] : 0.0;
              if (wupd && in) {
                stg_cs(wn + off, __fma_rn(-lp, uo, E[2 * KM2_VC + o]));
                if (!swd) stg_cs(swn + off, __fma_rn(-lp, E[4 * KM2_VC + o], E[3 * KM2_VC + o]));
              }
              double v = uo;
              if (upd) {
                v = in ? __fma_rn(mu, uo, E[KM2_VC + o]) : 0.0;
                if (in) u_io[off] = v;
              }
              p_b = __fma_rn(v, v, p_b);  // (u . u of the fast-path tiles: the math warps' epilogue)
            }
          }
          // this warp's reads of the stage are done (the arrival's release orders them before the next bulk copy)
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[cp.slot]);
          cp.next(nstage);
        }
        // the tile's u is in global memory: the math warps' epilogue may read it
        __syncwarp();
        if (lane == 0) mbar_arrive(&tile_done);
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(REG_MATH));
    // ---------------- math warps: DMMA m16n8k4, warp owns columns [8 NI warp, 8 NI (warp + 1)) of every tile
    const int g = lane >> 2, t = lane & 3;
    const int n0 = 8 * NI * warp;
    const double mu = st->mu;
    RingPos rp;
    for (int64_t jl = 0; jl < ntl; ++jl) {
      const int64_t k0 = (blockIdx.x + jl * gridDim.x) * KM_BM;
      double acc[4][NI][4];  // [m16 tile][n8 tile][fragment]
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[mi][ni][q] = 0.0;
      for (int s = 0; s < nchunk; ++s) {
        mbar_wait(&full[rp.slot], rp.phase);
        const double* S = ksm + rp.slot * sstride;
        const double* om = S + n0 + g;
        const double* U = S + KM2_OM + t * KM_XS + g;
#pragma unroll
        for (int kk = 0; kk < KM_OK / 4; ++kk) {
          const double* ob = om + (kk * 4 + t) * KM_OLD;
          double bq[NI];
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) bq[ni] = ob[8 * ni];
          const double* ua = U + kk * 4 * KM_XS;
          double a0[4], a1[4];
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) {
            a0[mi] = ua[16 * mi];
            a1[mi] = ua[16 * mi + 8];
          }
          if (upd) {  // u = pr + mu u_old (pcg.cpp:210), the value the side warps write
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) {
              a0[mi] = __fma_rn(mu, a0[mi], ua[KM2_VC + 16 * mi]);
              a1[mi] = __fma_rn(mu, a1[mi], ua[KM2_VC + 16 * mi + 8]);
            }
          }
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) dmma_16x8x4(acc[mi][ni], a0[mi], a1[mi], bq[ni]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[rp.slot]);
        rp.next(nstage);
      }
      // epilogue: acc[mi][ni] = rows 16 mi + (g, g + 8) x columns n0 + 8 ni + 2 t (+1); rows >= msig carry
      // zero variance; u . Sigma u with the tile's u from global memory (L2), one m16 row block's 16 values at a
      // time (one L2 round trip per row block)
      // the side warps have written this tile's u.  (They cannot be two tiles ahead: a tile has more chunks than the
      // ring has stages -- G > 128 -- and a stage is recycled only after every math warp released it.)
      if (!APPLY) mbar_wait(&tile_done, (uint32_t)(jl & 1));
      const bool tile_in = k0 + KM_BM <= ldm && n0 + 8 * NI <= G;
      // (measured and dropped: requesting the next row block's u before this one's stores -- 5.13 -> 5.37 ms; and
      // preparing each k-step's A operands one step ahead, peeking at the next stage with test_wait -- 5.9 ms)
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        double uv[NI][4];
        if (!APPLY) {
#pragma unroll
          for (int ni = 0; ni < NI; ++ni)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int c = n0 + 8 * ni + 2 * t + (q & 1);
              const int64_t grow = k0 + 16 * mi + g + 8 * (q >> 1);
              uv[ni][q] = (tile_in || (c < G && grow < ldm)) ? u_io[(int64_t)c * ldm + grow] : 0.0;
            }
        }
#pragma unroll
        for (int ni = 0; ni < NI; ++ni)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int c = n0 + 8 * ni + 2 * t + (q & 1);
            const int64_t grow = k0 + 16 * mi + g + 8 * (q >> 1);
            if (tile_in || (c < G && grow < ldm)) {
              const double o = grow < msig ? acc[mi][ni][q] : 0.0;
              stg_cs(out + (int64_t)c * ldm + grow, o);
              if (!APPLY) p_a = __fma_rn(uv[ni][q], o, p_a);
            }
          }
        if (!APPLY && fast && k0 + KM_BM <= ldm) {  // u . u of the tiles the side warps' fast path handled
#pragma unroll
          for (int ni = 0; ni < NI; ++ni)
#pragma unroll
            for (int q = 0; q < 4; ++q) p_b = __fma_rn(uv[ni][q], uv[ni][q], p_b);
        }
      }
    }
  }
  // (d, u.u) partials of this CTA, fixed order (pcg.cpp:144-145)
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    p_a += __shfl_xor_sync(FULL, p_a, o);
    p_b += __shfl_xor_sync(FULL, p_b, o);
  }
  if (lane == 0) {
    red[warp][0] = p_a;
    red[warp][1] = p_b;
  }
  __syncthreads();
  if (tid == 0 && !APPLY) {
    double a = 0.0, bb = 0.0;
    for (int w = 0; w < NTH / 32; ++w) {
      a += red[w][0];
      bb += red[w][1];
    }
    partials[blockIdx.x * 3 + 0] = a;
    partials[blockIdx.x * 3 + 1] = bb;
    partials[blockIdx.x * 3 + 2] = 0.0;
  }
}

// ------------------------------------------------------------------------------------------
// Fused pass C (fused_c knob, OFF by default; the k_kron_mma shapes with tile-contiguous Q): pr = Pi r (structured.cpp:307-317)
// with c = r.pr, r.r, pr.pr, AND Sigma pr = pr Omega on the FP64 tensor cores, in one sweep over 64-row tiles of
// all G blocks -- the Kronecker product hides under the Q stream.  Pass A then only needs the element-wise
// recurrences u = pr + mu u, Sigma u = Sigma pr + mu Sigma u (k_pass_a_ew): Sigma u is carried by recurrence
// instead of recomputed (the same value in exact arithmetic, rounded once more per iteration).
//   * element warps, per block b of a tile: the 64 x n_b sub-tile of Q_b (2-D TMA through the Q map, 16 KB
//     stages) and, per 8-block chunk, the 64 x 8 box of r; thread = row: pr = w (w r - Q_b t_b), then pr to
//     global and into the U chunk ring;
//   * math warps / Omega loader: as k_kron_mma, writing Sigma pr.
// Measured at c4: 18.3 ms for this pass + 3.2 ms for the element-wise pass A, against 10.9 + 6.9 ms for the
// separate passes.  Parity holds (test_fused_c_parity); the sweep is latency-bound -- two element warps per SM
// carry the Q_b t_b row products of all G blocks (the streaming pass C runs them on 256-512 threads per SM), and
// shared memory cannot hold the U ring, the Omega ring and the ~100 KB of Q in flight an SM needs for its share
// of HBM bandwidth at once.
constexpr int KC_EW = 2;                            // element warps of the fused pass C
constexpr int KC_NT = (KW_MATH + 1 + KC_EW) * 32;
constexpr int KC_QS = 5;                            // Q sub-tile stages (8 stages with 8 U slots / 2 Omega stages: slower)
constexpr int KC_RS = 3;                            // r box stages
constexpr int KC_OS = 3;                            // Omega slab stages
constexpr int KC_UR = 16;                           // U (pr) chunk slots
constexpr int KC_QT = 32 * KM_BM;                   // Q sub-tile doubles (32 columns x 64 rows)
constexpr int KC_RB = KM_OK * KM_BM;                // r box doubles (8 columns x 64 rows)
constexpr size_t kc_smem_bytes() {
  return (size_t)(KC_UR * KM_UC + KC_OS * KM_OK * KM_OLD + KC_QS * KC_QT + KC_RS * KC_RB) * sizeof(double);
}

__global__ void __launch_bounds__(KC_NT, 1) k_pass_c_mma(const __grid_constant__ CUtensorMap qmap,
                                                         const __grid_constant__ CUtensorMap vmap64, Geo g,
                                                         int64_t ntiles, const double* __restrict__ omegaT,
                                                         const double* __restrict__ t, const int64_t* __restrict__ qoff,
                                                         double* __restrict__ pr_out, double* __restrict__ spr_out,
                                                         double* partials, const SolveState* st, int gate) {
  if (gate == 1 && !st->active) return;
  extern __shared__ __align__(128) double ksm[];
  __shared__ __align__(8) uint64_t om_full[KC_OS], om_empty[KC_OS], q_full[KC_QS], q_empty[KC_QS], r_full[KC_RS],
      r_empty[KC_RS], uc_full[KC_UR], uc_empty[KC_UR];
  __shared__ double tsm[KC_EW][KM_OK][32];
  __shared__ double red[KC_NT / 32][3];
  double* const ucb = ksm;                                // [KC_UR][KM_OK][KM_XS]
  double* const omb = ucb + KC_UR * KM_UC;                // [KC_OS][KM_OK][KM_OLD]
  double* const qsb = omb + KC_OS * KM_OK * KM_OLD;       // [KC_QS][32][KM_BM]
  double* const rsb = qsb + KC_QS * KC_QT;                // [KC_RS][KM_OK][KM_BM]
  const int G = g.G;
  const int64_t ldm = g.ldm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nchunk = G / KM_OK;
  const int64_t ntl = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  if (tid == 0) {
    for (int i = 0; i < KC_OS; ++i) {
      mbar_init(&om_full[i], 1);
      mbar_init(&om_empty[i], KW_MATH);
    }
    for (int i = 0; i < KC_QS; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], KC_EW);
    }
    for (int i = 0; i < KC_RS; ++i) {
      mbar_init(&r_full[i], 1);
      mbar_init(&r_empty[i], KC_EW);
    }
    for (int i = 0; i < KC_UR; ++i) {
      mbar_init(&uc_full[i], KC_EW);
      mbar_init(&uc_empty[i], KW_MATH);
    }
    mbar_fence_init();
  }
  __syncthreads();
  double pc = 0.0, prr = 0.0, ppp = 0.0;
  if (warp == KW_MATH) {
    if (lane == 0) {  // Omega loader
      const uint32_t row_bytes = (uint32_t)(G * sizeof(double));
      RingPos w;
      int s = 0;
      for (int64_t q = 0; q < ntl * nchunk; ++q) {
        if (q >= KC_OS) mbar_wait(&om_empty[w.slot], w.phase ^ 1u);
        mbar_expect_tx(&om_full[w.slot], row_bytes * KM_OK);
        double* dst = omb + w.slot * KM_OK * KM_OLD;
        const double* src = omegaT + (int64_t)s * KM_OK * G;
#pragma unroll
        for (int r = 0; r < KM_OK; ++r) tma_load_1d(dst + r * KM_OLD, src + (int64_t)r * G, row_bytes, &om_full[w.slot]);
        w.next(KC_OS);
        if (++s == nchunk) s = 0;
      }
    }
  } else if (warp > KW_MATH) {
    // ---------------- element warps: thread = row (KC_EW * 32 == KM_BM), block by block
    const int ew = warp - KW_MATH - 1;
    const int row = ew * 32 + lane;
    const bool issuer = (ew == 0 && lane == 0);
    const int64_t totq = ntl * G, totr = ntl * nchunk;
    RingPos qi, ri;              // issue positions
    int64_t nq = 0, nr = 0, q_tile = blockIdx.x, r_tile = blockIdx.x;
    int q_b = 0, r_c = 0;
    auto issue_q = [&]() {
      if (nq >= KC_QS) mbar_wait(&q_empty[qi.slot], qi.phase ^ 1u);
      mbar_expect_tx(&q_full[qi.slot], (uint32_t)(KC_QT * sizeof(double)));
      const int64_t k0 = q_tile * KM_BM;
      const int nb = g.nb[q_b];
      const int64_t outer = (qoff[q_b] >> 8) + (k0 >> 8) * nb;  // 256-row tile (k0 / 256) of block q_b
      tma_load_2d(qsb + qi.slot * KC_QT, &qmap, (int)(k0 & 255), (int)outer, &q_full[qi.slot]);
      qi.next(KC_QS);
      ++nq;
      if (++q_b == G) {
        q_b = 0;
        q_tile += gridDim.x;
      }
    };
    auto issue_r = [&]() {
      if (nr >= KC_RS) mbar_wait(&r_empty[ri.slot], ri.phase ^ 1u);
      mbar_expect_tx(&r_full[ri.slot], (uint32_t)(KC_RB * sizeof(double)));
      tma_load_2d(rsb + ri.slot * KC_RB, &vmap64, (int)(r_tile * KM_BM), MV_R * G + r_c * KM_OK, &r_full[ri.slot]);
      ri.next(KC_RS);
      ++nr;
      if (++r_c == nchunk) {
        r_c = 0;
        r_tile += gridDim.x;
      }
    };
    if (issuer) {
      while (nq < KC_QS - 1 && nq < totq) issue_q();
      while (nr < KC_RS - 1 && nr < totr) issue_r();
    }
    RingPos qc, rc, up;
    // t of a chunk's 8 blocks, one value per lane per block, loaded one chunk ahead (no latency per block)
    double tv[KM_OK];
    auto load_t = [&](int c) {
#pragma unroll
      for (int bb = 0; bb < KM_OK; ++bb) {
        const int b = c * KM_OK + bb;
        tv[bb] = lane < g.nb[b] ? __ldg(t + g.p0[b] + lane) : 0.0;
      }
    };
    load_t(0);
    for (int64_t jl = 0; jl < ntl; ++jl) {
      const int64_t k0 = (blockIdx.x + jl * gridDim.x) * KM_BM;
      const int64_t k = k0 + row;
      for (int c = 0; c < nchunk; ++c) {
        if (issuer && nr < totr) issue_r();
#pragma unroll
        for (int bb = 0; bb < KM_OK; ++bb) tsm[ew][bb][lane] = tv[bb];
        __syncwarp();
        load_t(c + 1 < nchunk ? c + 1 : 0);  // the next chunk's t (wraps to the next tile's first chunk)
        mbar_wait(&r_full[rc.slot], rc.phase);
        if (jl * nchunk + c >= KC_UR) mbar_wait(&uc_empty[up.slot], up.phase ^ 1u);
        const double* R = rsb + rc.slot * KC_RB;
        double* U = ucb + up.slot * KM_UC;
        for (int bb = 0; bb < KM_OK; ++bb) {
          const int b = c * KM_OK + bb;
          if (issuer && nq < totq) issue_q();
          mbar_wait(&q_full[qc.slot], qc.phase);
          const double* Qs = qsb + qc.slot * KC_QT + row;
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            s0 = __fma_rn(Qs[(j + 0) * KM_BM], tsm[ew][bb][j + 0], s0);
            s1 = __fma_rn(Qs[(j + 1) * KM_BM], tsm[ew][bb][j + 1], s1);
            s2 = __fma_rn(Qs[(j + 2) * KM_BM], tsm[ew][bb][j + 2], s2);
            s3 = __fma_rn(Qs[(j + 3) * KM_BM], tsm[ew][bb][j + 3], s3);
          }
          const double proj = (s0 + s1) + (s2 + s3);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&q_empty[qc.slot]);
          qc.next(KC_QS);
          const double wgt = row_wgt(g, g.wts[b], g.wtc[b], k);
          const double rv = R[bb * KM_BM + row];
          const double pv = (rv * wgt - proj) * wgt;
          if (k < ldm) {
            stg_cs(pr_out + (int64_t)b * ldm + k, pv);
            pc += rv * pv;
            prr += rv * rv;
            ppp += pv * pv;
          }
          U[bb * KM_XS + row] = k < ldm ? pv : 0.0;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&r_empty[rc.slot]);
          mbar_arrive(&uc_full[up.slot]);
        }
        rc.next(KC_RS);
        up.next(KC_UR);
      }
    }
  } else {
    // ---------------- math warps: Sigma pr, as k_kron_mma
    const int gg = lane >> 2, tt = lane & 3;
    const int n0 = 32 * warp;
    RingPos rp, up;
    for (int64_t jl = 0; jl < ntl; ++jl) {
      const int64_t k0 = (blockIdx.x + jl * gridDim.x) * KM_BM;
      double acc[4][4][4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[mi][ni][q] = 0.0;
      for (int s = 0; s < nchunk; ++s) {
        mbar_wait(&uc_full[up.slot], up.phase);
        mbar_wait(&om_full[rp.slot], rp.phase);
        const double* om = omb + rp.slot * KM_OK * KM_OLD + n0 + gg;
        const double* U = ucb + up.slot * KM_UC + tt * KM_XS + gg;
#pragma unroll
        for (int kk = 0; kk < KM_OK / 4; ++kk) {
          const double* ob = om + (kk * 4 + tt) * KM_OLD;
          const double b0 = ob[0], b1 = ob[8], b2 = ob[16], b3 = ob[24];
          const double* ua = U + kk * 4 * KM_XS;
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) {
            const double a0 = ua[16 * mi], a1 = ua[16 * mi + 8];
            dmma_16x8x4(acc[mi][0], a0, a1, b0);
            dmma_16x8x4(acc[mi][1], a0, a1, b1);
            dmma_16x8x4(acc[mi][2], a0, a1, b2);
            dmma_16x8x4(acc[mi][3], a0, a1, b3);
          }
        }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&om_empty[rp.slot]);
          mbar_arrive(&uc_empty[up.slot]);
        }
        rp.next(KC_OS);
        up.next(KC_UR);
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int c = n0 + 8 * ni + 2 * tt + (q & 1);
            const int64_t grow = k0 + 16 * mi + gg + 8 * (q >> 1);
            if (c < G && grow < ldm)
              stg_cs(spr_out + (int64_t)c * ldm + grow, grow < g.msig ? acc[mi][ni][q] : 0.0);
          }
    }
  }
  // (c, r.r, pr.pr) partials of this CTA (pcg.cpp:157,165), fixed order
  double v[3] = {pc, prr, ppp};
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v[i] += __shfl_xor_sync(FULL, v[i], o);
  if (lane == 0) {
    red[warp][0] = v[0];
    red[warp][1] = v[1];
    red[warp][2] = v[2];
  }
  __syncthreads();
  if (tid == 0 && partials) {
    double a = 0.0, b = 0.0, c = 0.0;
    for (int w = 0; w < KC_NT / 32; ++w) {
      a += red[w][0];
      b += red[w][1];
      c += red[w][2];
    }
    partials[blockIdx.x * 3 + 0] = a;
    partials[blockIdx.x * 3 + 1] = b;
    partials[blockIdx.x * 3 + 2] = c;
  }
}

// Pass A of the fused schedule (element-wise, HBM-streaming over the slab columns): u = pr + mu u (pcg.cpp:210),
// Sigma u = Sigma pr + mu Sigma u (by linearity; pass C formed Sigma pr), the deferred w -= lambda u
// (pcg.cpp:151; sw_mode 1), d = u . Sigma u, u . u.  In the first iteration (no mu yet) u = pr already and
// Sigma u = Sigma pr.
__global__ void __launch_bounds__(NT) k_pass_a_ew(int64_t count, double* __restrict__ u, double* __restrict__ su,
                                                  const double* __restrict__ pr, const double* __restrict__ spr,
                                                  WBuf wbuf, double* partials, const SolveState* st) {
  if (!st->active) return;
  const bool upd = st->mu_pending != 0, wupd = st->upd_pending != 0;
  const double mu = st->mu, lp = st->lam_prev;
  const double* __restrict__ wc = wbuf.w[st->cur];
  double* __restrict__ wn = wbuf.w[st->nxt];
  double pd = 0.0, pu = 0.0;
  const int64_t n2 = count >> 1;  // double2 elements (count is even: ldm is a multiple of 32)
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 uo = reinterpret_cast<const double2*>(u)[i];
    const double2 sp = reinterpret_cast<const double2*>(spr)[i];
    double2 un = uo, sn = sp;
    if (upd) {
      const double2 pv = reinterpret_cast<const double2*>(pr)[i];
      const double2 so = reinterpret_cast<const double2*>(su)[i];
      un.x = pv.x + mu * uo.x;
      un.y = pv.y + mu * uo.y;
      sn.x = sp.x + mu * so.x;
      sn.y = sp.y + mu * so.y;
      reinterpret_cast<double2*>(u)[i] = un;
    }
    if (wupd) {
      const double2 wv = reinterpret_cast<const double2*>(wc)[i];
      double2 wo;
      wo.x = wv.x + (-lp) * uo.x;
      wo.y = wv.y + (-lp) * uo.y;
      reinterpret_cast<double2*>(wn)[i] = wo;
    }
    reinterpret_cast<double2*>(su)[i] = sn;
    pd += un.x * sn.x;
    pd += un.y * sn.y;
    pu += un.x * un.x;
    pu += un.y * un.y;
  }
  __shared__ double red[NT / 32 * 3];
  double v[3] = {pd, pu, 0.0};
  block_sum<3>(v, red);
  if (threadIdx.x == 0) {
    partials[blockIdx.x * 3 + 0] = v[0];
    partials[blockIdx.x * 3 + 1] = v[1];
    partials[blockIdx.x * 3 + 2] = 0.0;
  }
}

enum { SMODE_B = 0, SMODE_C = 1, SMODE_QT_R = 2, SMODE_QT_D = 3, SMODE_QT_V = 4, SMODE_DIAG = 5, SMODE_XS = 6,
       SMODE_BD = 7, SMODE_CD = 8 };
// SMODE_BD / SMODE_CD: passes B and C with the trace row's diagnostics folded in (diag_every = 1, xv_mode QR,
// narrow blocks; the reference fills aug_residual_norm / dual_feas_norm / rmse on every row, pcg.cpp:96-116):
//   BD: as B, plus z = w_b (y - sw_{i+1}), sw_{i+1} = sw_i - lambda su (written to zbuf), and the column partials
//       of Q'z (tpart2): est = R^-1 Q'z = X*'(y - sw_{i+1}) (recover, pcg.cpp:96-98), s_est = R est = Q'z;
//   CD: as C, plus |y - sw_{i+1} - X est|^2 = sum_k ((z_k - Q_k s_est) / w_b)^2 (partials2) and the column
//       partials of Q' w_{i+1}, w_{i+1} = w_i - lambda u (tpart3): X' w = R' Q' w / w_b (pcg.cpp:112).

struct StreamArgs {
  const double* Q;      // ld = ldm
  const double* X;      // ld = ldx (>= ldm, 16-byte aligned columns)
  int64_t ldx;
  const double* u;
  const double* su;
  double* wb[3];
  double* swb[3];
  double* r;
  double* pr;           // SMODE_C output
  double* out;          // SMODE_XS output
  const double* y;
  int64_t ldy;
  const double* vin;    // SMODE_QT_V input
  const double* vec;    // per-block n-vector: v / s (B), t (C, XS), est (DIAG)
  double* tpart;        // column partials [(p0 + j) * nch + ch]
  double* partials;     // per-CTA dot partials (C: 3, DIAG: 1)
  double* zbuf;         // BD: z = w_b (y - sw_{i+1}) out; CD: in
  const double* vec2;   // CD: s_est = Q'z per block (the reduced tpart2)
  double* tpart2;       // BD: Q'z column partials
  double* tpart3;       // CD: Q' w_{i+1} column partials
  double* partials2;    // CD: per-CTA residual partial
  int xv_from_x, sel_best, gate;
  int T, S, nmax;
  int qdiag;            // SMODE_DIAG from Q instead of X (xv_mode QR): X est = Q s / w with s = R est, and the
                        // column partials are Q' w (X' w = R' Q' w / w, k_rt_apply)
  int qtiled;           // Q stored tile-contiguous (qtile-row tiles per block, column-major inside)
  int qtile;            // rows per Q tile (256 for narrow blocks, 64 for the wide blocks' tiled copy)
  const int64_t* qoff;  // [G] offset of Q_b (tiled layout)
  int64_t stage_doubles;
};

template <int MODE>
__device__ __forceinline__ int stream_nmat(const StreamArgs& a) {
  return MODE == SMODE_B ? 1 + a.xv_from_x : 1;
}
template <int MODE>
__host__ __device__ constexpr int stream_nvec() {
  return MODE == SMODE_B ? 2 : MODE == SMODE_DIAG ? 4 : MODE == SMODE_QT_D ? 2 : MODE == SMODE_XS ? 0
         : MODE == SMODE_BD ? 4 : MODE == SMODE_CD ? 4 : 1;
}

template <int MODE, bool FUSE>
__global__ void __launch_bounds__(NT) k_stream(Geo g, StreamArgs a, const SolveState* st) {
  if (a.gate == 1 && !st->active) return;
  if (a.gate == 2 && !st->diag_now) return;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bars[4];
  __shared__ double red[NT / 32 * 4];
  __shared__ double fred[(FUSE && (MODE != SMODE_C && MODE != SMODE_XS)) ? NT : 1];
  __shared__ double tv2[MODE == SMODE_CD ? 128 : 1];
  __shared__ double pdot[FUSE ? 1 : NT];  // wide blocks: partial row dots [P][T]
  const int S = a.S, T = a.T;
  double* xs = sm + (int64_t)S * a.stage_doubles;
  // per-item n-vector slice (nmax <= 128 on this path): a static shared array, so the row dots read it
  // with immediate shared-memory offsets
  __shared__ double tv[128];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nmat = stream_nmat<MODE>(a);
  constexpr int NV = stream_nvec<MODE>();
  const int64_t items = (int64_t)g.G * g.nch;

  double lam = 0.0, lp = 0.0;  // lp: lambda of a still-pending w / sw update (diagnostics apply it on the fly)
  int cur = 0, sel = 0;
  if (MODE == SMODE_B || MODE == SMODE_BD || MODE == SMODE_CD) lam = st->lambda;
  if (MODE == SMODE_DIAG || MODE == SMODE_BD || MODE == SMODE_CD) cur = st->cur;
  if (MODE == SMODE_QT_D) sel = a.sel_best ? (st->term == T_CONVERGED ? st->cur : st->best) : st->cur;
  if ((MODE == SMODE_DIAG || MODE == SMODE_QT_D) && st && st->upd_pending) lp = st->lam_prev;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    mbar_fence_init();
  }
  {
    // the narrow-block sweep reads all 32 column slots of a stage, and the wide-block column pass reads whole
    // tiles (the rows of a partial tile meet x = 0): start from finite contents
    for (int64_t i = tid; i < (int64_t)S * a.stage_doubles; i += NT) sm[i] = 0.0;
    fence_proxy_async_smem();  // generic writes ordered before the first TMA writes into the ring
  }
  __syncthreads();

  // tile iterator (item = blockIdx.x + j * gridDim.x; tiles of T rows inside the item's chunk)
  auto item_rows = [&](int64_t item, int64_t& k0, int64_t& k1) {
    const int ch = (int)(item % g.nch);
    k0 = (int64_t)ch * g.CH;
    k1 = (k0 + g.CH < g.ldm) ? k0 + g.CH : g.ldm;
  };
  // producer position: the current item's block / rows are cached (one division per item, not per tile)
  int64_t p_item = blockIdx.x, p_tile = 0, p_k0 = 0, p_k1 = 0, p_p0 = 0;
  int p_b = 0, p_nb = 0;
  auto p_load = [&]() {
    if (p_item >= items) return;
    item_rows(p_item, p_k0, p_k1);
    p_b = (int)(p_item / g.nch);
    p_nb = g.nb[p_b];
    p_p0 = g.p0[p_b];
  };
  p_load();
  auto issue = [&](int stage) {
    // warp 0 only; advances the producer iterator
    if (p_item >= items) return;
    const int64_t k0 = p_k0, k1 = p_k1;
    const int64_t kb = k0 + p_tile * T;
    const int rows = (int)((k1 - kb) < T ? (k1 - kb) : T);
    const int b = p_b;
    const int nb = p_nb;
    const int64_t p0 = p_p0;
    const uint32_t seg = (uint32_t)rows * 8u;
    // tile-contiguous Q with T == 256: the whole tile (padded to 256 rows) is ONE contiguous region,
    // moved as 4 bulk copies; otherwise one copy per column segment
    const bool qbig = (MODE != SMODE_DIAG || a.qdiag) && a.qtiled && T == a.qtile;
    const int nq = qbig ? 4 : nb;
    const int nseg = nq + (nmat - 1) * nb + NV;
    const uint32_t qpiece = (uint32_t)(T * nb * 8 / 4);
    const uint32_t total = (qbig ? 4u * qpiece : seg * (uint32_t)nb) + seg * (uint32_t)((nmat - 1) * nb + NV);
    double* base = sm + (int64_t)stage * a.stage_doubles;
    if (lane == 0) mbar_expect_tx(&bars[stage], total);
    __syncwarp();
    for (int q = lane; q < nseg; q += 32) {
      const double* src;
      double* dst;
      uint32_t bytes = seg;
      if (q < nq) {  // first matrix: Q (X for DIAG)
        if (MODE == SMODE_DIAG && !a.qdiag) {
          src = a.X + (p0 + q) * a.ldx + kb;
          dst = base + (int64_t)q * T;
        } else if (qbig) {
          src = a.Q + a.qoff[b] + (kb / a.qtile) * (int64_t)(a.qtile * nb) + (int64_t)q * (qpiece / 8);
          dst = base + (int64_t)q * (qpiece / 8);
          bytes = qpiece;
        } else if (a.qtiled) {
          src = a.Q + a.qoff[b] + (kb / a.qtile) * (int64_t)(a.qtile * nb) + (int64_t)q * a.qtile + (kb % a.qtile);
          dst = base + (int64_t)q * T;
        } else {
          src = a.Q + (p0 + q) * g.ldm + kb;
          dst = base + (int64_t)q * T;
        }
      } else if (q < nq + (nmat - 1) * nb) {  // second matrix: X (pass B, xv_mode X)
        src = a.X + (p0 + (q - nq)) * a.ldx + kb;
        dst = base + (int64_t)(nb + (q - nq)) * T;
      } else {
        const int v = q - nq - (nmat - 1) * nb;
        const int64_t vo = (int64_t)b * g.ldm + kb;
        const double* vb = nullptr;
        if (MODE == SMODE_B) vb = v == 0 ? a.su : a.r;
        else if (MODE == SMODE_BD) vb = v == 0 ? a.su : v == 1 ? a.r : v == 2 ? a.swb[cur] : nullptr;
        else if (MODE == SMODE_CD) vb = v == 0 ? a.r : v == 1 ? a.zbuf : v == 2 ? a.wb[cur] : a.u;
        else if (MODE == SMODE_C || MODE == SMODE_QT_R) vb = a.r;
        else if (MODE == SMODE_QT_V) vb = a.vin;
        else if (MODE == SMODE_QT_D) vb = v == 0 ? a.swb[sel] : a.su;
        else if (MODE == SMODE_DIAG) vb = v == 0 ? a.wb[cur] : v == 1 ? a.swb[cur] : v == 2 ? a.u : a.su;
        src = (MODE == SMODE_BD && v == 3) ? a.y + (int64_t)b * a.ldy + kb : vb + vo;  // y: ld ldy >= ldm (h->fold)
        dst = base + (int64_t)(nmat * nb) * T + (int64_t)v * T;
      }
      tma_load_1d(dst, src, bytes, &bars[stage]);
    }
    if (++p_tile * T >= k1 - k0) {
      p_tile = 0;
      p_item += gridDim.x;
      p_load();
    }
  };
  if (warp == 0)
    for (int s = 0; s < S; ++s) issue(s);

  double pc = 0.0, prr = 0.0, ppp = 0.0, rsum = 0.0;
  constexpr int MAXC = 16;  // columns per warp (n_b <= 128 on this path)
  constexpr bool COLS = (MODE != SMODE_C && MODE != SMODE_XS);
  constexpr bool COLS2 = (MODE == SMODE_BD);  // a second column-partial set (Q'z)
  int64_t it_count = 0;
  for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
    int64_t k0, k1;
    item_rows(item, k0, k1);
    const int b = (int)(item / g.nch);
    const int ch = (int)(item % g.nch);
    const int nb = g.nb[b];
    const int64_t p0 = g.p0[b];
    const double wz = g.wts[b], wc = g.wtc[b];
    const double iwz = 1.0 / wz, iwc = 1.0 / wc;  // Q-side X v = Q (R v) / w (exact when w = 1)
    const int64_t vbase = (int64_t)b * g.ldm;
    // tv holds >= 32 entries (zero past n_b): the fused row dots read all 32
    for (int j = tid; j < (nb > 32 ? nb : 32); j += NT)
      if (MODE == SMODE_B || MODE == SMODE_C || MODE == SMODE_XS || MODE == SMODE_DIAG || MODE == SMODE_BD ||
          MODE == SMODE_CD) {
        tv[j] = (j < nb) ? a.vec[p0 + j] : 0.0;
        if (MODE == SMODE_CD) tv2[j] = (j < nb) ? a.vec2[p0 + j] : 0.0;
      }
    __syncthreads();
    // column partials live in registers across the item's tiles: lane partial of column warp + 8 c
    double acc[MAXC];
#pragma unroll
    for (int q = 0; q < MAXC; ++q) acc[q] = 0.0;
    double facc[(FUSE && COLS) ? 32 : 1];
#pragma unroll
    for (int j = 0; j < ((FUSE && COLS) ? 32 : 1); ++j) facc[j] = 0.0;
    double facc2[(FUSE && COLS2) ? 32 : 1];
#pragma unroll
    for (int j = 0; j < ((FUSE && COLS2) ? 32 : 1); ++j) facc2[j] = 0.0;
    for (int64_t kb = k0; kb < k1; kb += T, ++it_count) {
      const int stage = (int)(it_count % S);
      const int rows = (int)((k1 - kb) < T ? (k1 - kb) : T);
      mbar_wait(&bars[stage], (uint32_t)((it_count / S) & 1));
      const double* base = sm + (int64_t)stage * a.stage_doubles;
      const double* M0 = base;                                 // Q (X for DIAG)
      const double* M1 = base + (int64_t)nb * T;               // X (pass B, xv_mode X)
      const double* V = base + (int64_t)(nmat * nb) * T;       // vectors
      if constexpr (FUSE) {
        // narrow blocks (n_b <= 32): the row of the tile's matrix lives in registers; the row work and
        // the column partials (acc_j += A[k, j] x_k) happen in one sweep -- no second phase, no extra
        // barrier; the per-lane accumulators are transpose-reduced once per item.  All 32 columns are
        // read unconditionally (immediate shared-memory offsets, no per-column branch): columns past
        // n_b hold finite stale data (the ring is zero-filled at launch and only ever receives finite
        // Q / vector tiles) and meet tv[j] = 0 in the row dot, and their column partials are dropped.
        // Row dots and column partials are fixed-shape sums (not the reference's order anyway), so
        // they use fused multiply-adds.
        for (int t = tid; t < rows; t += NT) {
          const int64_t k = kb + t;
          const int64_t vo = vbase + k;
          const bool zrow = k < g.msig;
          const double wgt = zrow ? wz : wc, iwgt = zrow ? iwz : iwc;
          constexpr bool ROWREG = (MODE != SMODE_BD && MODE != SMODE_CD);  // the folded modes read Q from smem
          double arow[ROWREG ? 32 : 1];
          if constexpr (ROWREG) {
#pragma unroll
            for (int j = 0; j < 32; ++j) arow[j] = M0[(int64_t)j * T + t];
          }
          // row dot from shared memory (the folded modes: two / three column-partial sets leave no room for
          // the row in registers)
          auto sdot = [&](const double* tvp) {
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              s0 = __fma_rn(M0[(int64_t)(j + 0) * T + t], tvp[j + 0], s0);
              s1 = __fma_rn(M0[(int64_t)(j + 1) * T + t], tvp[j + 1], s1);
              s2 = __fma_rn(M0[(int64_t)(j + 2) * T + t], tvp[j + 2], s2);
              s3 = __fma_rn(M0[(int64_t)(j + 3) * T + t], tvp[j + 3], s3);
            }
            return (s0 + s1) + (s2 + s3);
          };
          (void)sdot;
          auto rdot = [&]() {
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              s0 = __fma_rn(arow[j + 0], tv[j + 0], s0);
              s1 = __fma_rn(arow[j + 1], tv[j + 1], s1);
              s2 = __fma_rn(arow[j + 2], tv[j + 2], s2);
              s3 = __fma_rn(arow[j + 3], tv[j + 3], s3);
            }
            return (s0 + s1) + (s2 + s3);
          };
          double x = 0.0, x2 = 0.0;
          if (MODE == SMODE_BD) {
            const double suv = V[t], rv = V[T + t], swv = V[2 * T + t];
            const double xv = sdot(tv) * iwgt;
            const double rn = rv - lam * (suv + xv);
            a.r[vo] = rn;
            x = rn * wgt;
            const double yv = (k < g.M) ? V[3 * T + t] : 0.0;
            x2 = (yv - (swv + (-lam) * suv)) * wgt;
            a.zbuf[vo] = x2;
          } else if (MODE == SMODE_CD) {
            const double proj = sdot(tv);
            const double rv = V[t];
            const double pv = (rv * wgt - proj) * wgt;
            a.pr[vo] = pv;
            pc += rv * pv;
            prr += rv * rv;
            ppp += pv * pv;
            asm volatile("" ::: "memory");  // re-read the row from shared memory (keeps it out of registers)
            const double res = (V[T + t] - sdot(tv2)) * iwgt;
            if (k < g.M) rsum += res * res;
            x = V[2 * T + t] + (-lam) * V[3 * T + t];  // w_{i+1}
          } else if (MODE == SMODE_B) {
            const double suv = V[t], rv = V[T + t];
            double xv = 0.0;
            if (a.xv_from_x) {
              if (k < g.M)
                for (int j = 0; j < nb; ++j) xv = xv + M1[(int64_t)j * T + t] * tv[j];
            } else {
              xv = rdot() * iwgt;
            }
            const double rn = rv - lam * (suv + xv);
            a.r[vo] = rn;
            x = rn * wgt;
          } else if (MODE == SMODE_C || MODE == SMODE_XS) {
            const double proj = rdot();
            if (MODE == SMODE_XS) {
              a.out[vo] = proj * wgt;
            } else {
              const double rv = V[t];
              const double pv = (rv * wgt - proj) * wgt;
              a.pr[vo] = pv;
              pc += rv * pv;
              prr += rv * rv;
              ppp += pv * pv;
            }
          } else if (MODE == SMODE_QT_R || MODE == SMODE_QT_V) {
            x = V[t] * wgt;
          } else if (MODE == SMODE_QT_D) {
            const double yv = (k < g.M) ? a.y[(int64_t)b * a.ldy + k] : 0.0;
            x = (yv - (V[t] + (-lp) * V[T + t])) * wgt;
          } else {  // SMODE_DIAG
            const double xe = (k < g.M) ? (a.qdiag ? rdot() * iwgt : rdot()) : 0.0;
            const double yv = (k < g.M) ? a.y[(int64_t)b * a.ldy + k] : 0.0;
            const double res = yv - ((V[T + t] + (-lp) * V[3 * T + t]) + xe);
            if (k < g.M) rsum += res * res;
            x = V[t] + (-lp) * V[2 * T + t];
          }
          if constexpr (COLS && ROWREG) {
#pragma unroll
            for (int j = 0; j < 32; ++j) facc[j] = __fma_rn(arow[j], x, facc[j]);
          }
          if constexpr (COLS && !ROWREG) {
            asm volatile("" ::: "memory");  // re-read the row from shared memory (keeps it out of registers)
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const double q = M0[(int64_t)j * T + t];
              facc[j] = __fma_rn(q, x, facc[j]);
              if constexpr (COLS2) facc2[j] = __fma_rn(q, x2, facc2[j]);
            }
          }
        }
        __syncthreads();  // the stage is free
        if (warp == 0) issue(stage);
        continue;
      }
      // ---- phase 1: row work (thread per row).  Q-side row sums use 4 independent chains (their
      // inputs come from tree reductions anyway); the X v row sum of xv_mode X stays sequential in j
      // (bitwise the reference's DenseMatrix::apply, dense_matrix.cpp:69-79).
      auto qdot = [&](const double* Mrow) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int j = 0;
        for (; j + 4 <= nb; j += 4) {
          s0 = s0 + Mrow[(int64_t)(j + 0) * T] * tv[j + 0];
          s1 = s1 + Mrow[(int64_t)(j + 1) * T] * tv[j + 1];
          s2 = s2 + Mrow[(int64_t)(j + 2) * T] * tv[j + 2];
          s3 = s3 + Mrow[(int64_t)(j + 3) * T] * tv[j + 3];
        }
        for (; j < nb; ++j) s0 = s0 + Mrow[(int64_t)j * T] * tv[j];
        return (s0 + s1) + (s2 + s3);
      };
      // wide blocks with T < NT: every thread helps with the Q-side row dots -- thread (p, r) = (tid / T, tid % T)
      // sums columns [p nb / P, (p + 1) nb / P) of row r (consecutive rows per warp: conflict-free), the P
      // partials are then added in p order; with one thread per row a 118-long dot on 64 of 256 threads was the
      // pass's critical path
      constexpr bool QROW = (MODE == SMODE_B || MODE == SMODE_C || MODE == SMODE_XS || MODE == SMODE_DIAG);
      const int P = NT / T;
      const bool coop = QROW && P > 1 && !(MODE == SMODE_B && a.xv_from_x) && !(MODE == SMODE_DIAG && !a.qdiag);
      if (coop) {
        const int pp = tid / T, rr = tid - pp * T;
        const int j0 = pp * nb / P, j1 = (pp + 1) * nb / P;
        double s0 = 0.0, s1 = 0.0;
        if (rr < rows) {
          const double* Mrow = M0 + rr;
          int j = j0;
          for (; j + 2 <= j1; j += 2) {
            s0 = __fma_rn(Mrow[(int64_t)(j + 0) * T], tv[j + 0], s0);
            s1 = __fma_rn(Mrow[(int64_t)(j + 1) * T], tv[j + 1], s1);
          }
          if (j < j1) s0 = __fma_rn(Mrow[(int64_t)j * T], tv[j], s0);
        }
        pdot[tid] = s0 + s1;
        __syncthreads();
      }
      auto rowq = [&](int t) {
        if (!coop) return qdot(M0 + t);
        double s = pdot[t];
        for (int q = 1; q < P; ++q) s += pdot[q * T + t];
        return s;
      };
      for (int t = tid; t < rows; t += NT) {
        const int64_t k = kb + t;
        const int64_t vo = vbase + k;
        const bool zrow = k < g.msig;
        const double wgt = zrow ? wz : wc, iwgt = zrow ? iwz : iwc;
        if (MODE == SMODE_B) {
          // (w / sw updates are deferred to the next pass A)
          const double suv = V[t], rv = V[T + t];
          double xv = 0.0;
          if (a.xv_from_x) {
            if (k < g.M)
              for (int j = 0; j < nb; ++j) xv = xv + M1[(int64_t)j * T + t] * tv[j];
          } else {
            xv = rowq(t) * iwgt;
          }
          const double rn = rv - lam * (suv + xv);
          a.r[vo] = rn;
          xs[t] = rn * wgt;
        } else if (MODE == SMODE_C || MODE == SMODE_XS) {
          const double proj = rowq(t);
          if (MODE == SMODE_XS) {
            a.out[vo] = proj * wgt;
          } else {
            const double rv = V[t];
            const double pv = (rv * wgt - proj) * wgt;
            a.pr[vo] = pv;
            pc += rv * pv;
            prr += rv * rv;
            ppp += pv * pv;
          }
        } else if (MODE == SMODE_QT_R || MODE == SMODE_QT_V) {
          xs[t] = V[t] * wgt;
        } else if (MODE == SMODE_QT_D) {
          const double yv = (k < g.M) ? a.y[(int64_t)b * a.ldy + k] : 0.0;
          const double swv = V[t] + (-lp) * V[T + t];  // sw_{i+1} = sw_i - lambda_i su_i when pending
          xs[t] = (yv - swv) * wgt;
        } else {  // SMODE_DIAG
          const double xe = (k < g.M) ? (a.qdiag ? rowq(t) * iwgt : rowq(t)) : 0.0;
          const double yv = (k < g.M) ? a.y[(int64_t)b * a.ldy + k] : 0.0;
          const double swv = V[T + t] + (-lp) * V[3 * T + t];
          const double res = yv - (swv + xe);
          if (k < g.M) rsum += res * res;
          xs[t] = V[t] + (-lp) * V[2 * T + t];
        }
      }
      // ---- phase 2: column partials acc_j += sum_rows A[k, j] x_k (warp per column, lanes over rows).  The lane's
      // x values are hoisted into registers and the row loop is unrolled for the tile height (rows of a partial
      // last tile carry x = 0, set below, so no per-row bound check); fused multiply-adds (tree sums anyway)
      if (COLS) {
        for (int t = rows + tid; t < T; t += NT) xs[t] = 0.0;
        __syncthreads();
        auto cols = [&](auto rpl_tag) {
          constexpr int RPL = decltype(rpl_tag)::value;
          double xr[RPL];
#pragma unroll
          for (int i = 0; i < RPL; ++i) xr[i] = xs[lane + 32 * i];
#pragma unroll
          for (int q = 0; q < MAXC; ++q) {
            const int j = warp + (NT / 32) * q;
            if (j < nb) {
              const double* Mj = M0 + (int64_t)j * T + lane;
              double s = acc[q];
#pragma unroll
              for (int i = 0; i < RPL; ++i) s = __fma_rn(Mj[32 * i], xr[i], s);
              acc[q] = s;
            }
          }
        };
        if (T == 64) cols(std::integral_constant<int, 2>{});
        else if (T == 128) cols(std::integral_constant<int, 4>{});
        else if (T == 256) cols(std::integral_constant<int, 8>{});
        else cols(std::integral_constant<int, 1>{});
      }
      __syncthreads();  // the stage (and xs) are free
      if (warp == 0) issue(stage);
    }
    if constexpr (FUSE && COLS) {
      // transpose-reduce the 32 per-lane column partials, then the 8 warps in order
      double* tp = (MODE == SMODE_CD) ? a.tpart3 : a.tpart;
      warp_transpose_reduce<32>(facc);
      fred[warp * 32 + lane] = facc[0];
      __syncthreads();
      if (tid < nb) {
        double s = 0.0;
        for (int w = 0; w < NT / 32; ++w) s += fred[w * 32 + tid];
        tp[(p0 + tid) * g.nch + ch] = s;
      }
      __syncthreads();
      if constexpr (COLS2) {
        warp_transpose_reduce<32>(facc2);
        fred[warp * 32 + lane] = facc2[0];
        __syncthreads();
        if (tid < nb) {
          double s = 0.0;
          for (int w = 0; w < NT / 32; ++w) s += fred[w * 32 + tid];
          a.tpart2[(p0 + tid) * g.nch + ch] = s;
        }
        __syncthreads();
      }
    } else if (COLS) {
#pragma unroll
      for (int q = 0; q < MAXC; ++q) {
        const int j = warp + (NT / 32) * q;
        if (j < nb) {  // warp-uniform
          double s = acc[q];
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
          if (lane == 0) a.tpart[(p0 + j) * g.nch + ch] = s;
        }
      }
    }
  }
  if (MODE == SMODE_CD) {
    double v[4] = {pc, prr, ppp, rsum};
    block_sum<4>(v, red);
    if (tid == 0) {
      a.partials[blockIdx.x * 3 + 0] = v[0];
      a.partials[blockIdx.x * 3 + 1] = v[1];
      a.partials[blockIdx.x * 3 + 2] = v[2];
      a.partials2[blockIdx.x] = v[3];
    }
  }
  if (MODE == SMODE_C || MODE == SMODE_DIAG) {
    double v[3] = {MODE == SMODE_C ? pc : rsum, prr, ppp};
    block_sum<3>(v, red);
    if (tid == 0) {
      if (MODE == SMODE_C) {
        a.partials[blockIdx.x * 3 + 0] = v[0];
        a.partials[blockIdx.x * 3 + 1] = v[1];
        a.partials[blockIdx.x * 3 + 2] = v[2];
      } else {
        a.partials[blockIdx.x] = v[0];
      }
    }
  }
}

// Tiled copy of a column-major Q (ld ldm) for the wide blocks' streaming passes: block b, rows [TQ k, TQ k + TQ)
// become one contiguous TQ x n_b column-major tile at qtoff[b] + k TQ n_b (rows past ldm are zero).
__global__ void k_q_relayout(const double* __restrict__ Q, int64_t ldm, const int64_t* __restrict__ p0,
                             const int* __restrict__ nb, const int64_t* __restrict__ qtoff, int TQ, int G,
                             double* __restrict__ Qt) {
  const int b = blockIdx.y;
  if (b >= G) return;
  const int n = nb[b];
  const int64_t ntile = (ldm + TQ - 1) / TQ;
  const int64_t total = ntile * TQ * n;
  const double* src = Q + p0[b] * ldm;
  double* dst = Qt + qtoff[b];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / ((int64_t)TQ * n), rem = i - k * TQ * n;
    const int j = (int)(rem / TQ), r = (int)(rem - (int64_t)j * TQ);
    const int64_t row = k * TQ + r;
    dst[i] = row < ldm ? src[(int64_t)j * ldm + row] : 0.0;
  }
}

// Sum the chunk partials of every parameter (one warp per parameter, fixed order) -> out[n].
__global__ void k_reduce_t(const double* tpart, int64_t n, int nch, double* out, const SolveState* st,
                           int gate) {
  if (gate == 1 && !st->active) return;
  if (gate == 2 && !st->diag_now) return;
  const int lane = threadIdx.x & 31;
  const int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= n) return;
  double s = 0.0;
  for (int c = lane; c < nch; c += 32) s += tpart[j * nch + c];
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
  if (lane == 0) out[j] = s;
}

// Multi-rank: t = sum over ranks (in rank order) of the gathered local sums t_all[P][n].
__global__ void k_sum_ranks(const double* t_all, int nranks, int64_t n, double* out, const SolveState* st, int gate) {
  if (gate == 1 && !st->active) return;
  if (gate == 2 && !st->diag_now) return;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < nranks; ++r) s += t_all[(int64_t)r * n + j];
    out[j] = s;
  }
}

// Multi-rank TSQR: scatter the gathered per-rank top R factors (rall[P][sum n_b^2], each block
// column-major n_b x n_b at r0_b) into the per-block stacks [R_0; ...; R_{P-1}] (P n_b x n_b, ld P n_b).
__global__ void k_stack_r(const double* rall, int nranks, int64_t rtot, int G, const int* nb, const int64_t* r0,
                          const int64_t* stack_off, double* stacks) {
  const int b = blockIdx.x;
  if (b >= G) return;
  const int n = nb[b];
  const int64_t ld = (int64_t)nranks * n;
  double* S = stacks + stack_off[b];
  for (int64_t idx = threadIdx.x; idx < (int64_t)nranks * n * n; idx += blockDim.x) {
    const int r = (int)(idx / ((int64_t)n * n));
    const int64_t e = idx - (int64_t)r * n * n;
    const int j = (int)(e / n), i = (int)(e - (int64_t)j * n);
    S[(int64_t)j * ld + (int64_t)r * n + i] = rall[(int64_t)r * rtot + r0[b] + e];
  }
}

// Upper-triangular back substitution R x = b per block (linalg.cpp:130-136) or R' x = b
// (linalg.cpp:137-145), one thread per block, the reference's loop order.
__device__ __forceinline__ void tri_solve_dev(int n, const double* R, double* x, bool transpose) {
  if (!transpose) {
    for (int i = n - 1; i >= 0; --i) {
      double s = x[i];
      for (int j = i + 1; j < n; ++j) s -= R[i + (int64_t)j * n] * x[j];
      x[i] = s / R[i + (int64_t)i * n];
    }
  } else {
    for (int i = 0; i < n; ++i) {
      double s = x[i];
      for (int j = 0; j < i; ++j) s -= R[j + (int64_t)i * n] * x[j];
      x[i] = s / R[i + (int64_t)i * n];
    }
  }
}

// v update (pcg.cpp:208-209): v = R^-1 t + mu v (xv_mode X) or s = t + mu s (QR).
// mode 0: continue-gated iteration update; mode 1: init v = R^-1 t (X) / s = t (QR);
// mode 2: plain out = R^-1 t (recover / est / probes); mode 3: out = R'^-1 t (apply_xstar).
__global__ void k_vupdate(Geo g, const double* R, double* t, double* vs, int xv_from_x, int mode,
                          const SolveState* st) {
  if (mode == 0 && (!st->active || !st->cont)) return;
  if (mode == 2 && st && !st->diag_now) return;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.G) return;
  const int nb = g.nb[b];
  const int64_t p0 = g.p0[b];
  double* tb = t + p0;
  if (mode == 3) { tri_solve_dev(nb, R + g.r0[b], tb, true); return; }
  if (mode == 2 || xv_from_x) tri_solve_dev(nb, R + g.r0[b], tb, false);
  if (mode == 2) return;
  if (mode == 1) {
    for (int j = 0; j < nb; ++j) vs[p0 + j] = tb[j];
  } else {
    const double mu = st->mu;
    for (int j = 0; j < nb; ++j) vs[p0 + j] = tb[j] + mu * vs[p0 + j];
  }
}

// Q-side diagnostics (xv_mode QR, X not read): xtw_b = R_b' t_b / w_b, i.e. X_b' w from t_b = Q_b' w
// (X_b = Q_b R_b / w_b); gated on the diagnostics row like k_vupdate mode 2.
__global__ void k_rt_apply(Geo g, const double* R, const double* t, double* out, const SolveState* st) {
  if (st && !st->diag_now) return;
  const int b = blockIdx.y;
  const int nb = g.nb[b];
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nb) return;
  const int64_t p0 = g.p0[b];
  const double* Rb = R + g.r0[b];
  double s = 0.0;
  for (int i = 0; i <= j; ++i) s += Rb[i + (int64_t)j * nb] * t[p0 + i];
  out[p0 + j] = s / g.wts[b];
}

// dst = src (n entries), gated on the diagnostics row when st is given
__global__ void k_copy_gated(double* dst, const double* src, int64_t n, const SolveState* st) {
  if (st && !st->diag_now) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// ------------------------------------------------------------------------------------------
// Row pass: out_k = w_b (w_b in_k - sum_j Q[k,j] t_j)   (pi_impl, structured.cpp:307-317), or
// out_k = w_b (sum_j Q[k,j] t_j)                         (xstar_impl, structured.cpp:330-340).
// Partials per CTA (pi mode): [0] = r.pr, [1] = r.r, [2] = pr.pr   (pcg.cpp:157,165).
__global__ void __launch_bounds__(NT) k_rowpass(Geo g, const double* Q, const double* t, const double* in,
                                                double* out, double* partials, int xstar_mode,
                                                const SolveState* st) {
  if (st && !st->active) return;
  __shared__ double ts[512];
  __shared__ double red[NT / 32 * 3];
  const int64_t items = (int64_t)g.G * g.nch;
  double pc = 0.0, prr = 0.0, ppp = 0.0;
  for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const int b = (int)(item / g.nch);
    const int ch = (int)(item % g.nch);
    const int nb = g.nb[b];
    const int64_t p0 = g.p0[b];
    const double wz = g.wts[b], wc = g.wtc[b];
    __syncthreads();
    for (int j = threadIdx.x; j < nb; j += NT) ts[j] = t[p0 + j];
    __syncthreads();
    const double* Qb = Q + p0 * g.ldm;
    const int64_t k0 = (int64_t)ch * g.CH;
    const int64_t k1 = (k0 + g.CH < g.ldm) ? k0 + g.CH : g.ldm;
    const int64_t vo = (int64_t)b * g.ldm;
    for (int64_t k = k0 + threadIdx.x; k < k1; k += NT) {
      double proj = 0.0;
      int j = 0;
      for (; j + 4 <= nb; j += 4) {
        const double q0 = Qb[(int64_t)(j + 0) * g.ldm + k];
        const double q1 = Qb[(int64_t)(j + 1) * g.ldm + k];
        const double q2 = Qb[(int64_t)(j + 2) * g.ldm + k];
        const double q3 = Qb[(int64_t)(j + 3) * g.ldm + k];
        proj = proj + q0 * ts[j + 0];
        proj = proj + q1 * ts[j + 1];
        proj = proj + q2 * ts[j + 2];
        proj = proj + q3 * ts[j + 3];
      }
      for (; j < nb; ++j) proj = proj + Qb[(int64_t)j * g.ldm + k] * ts[j];
      const double wgt = row_wgt(g, wz, wc, k);
      if (xstar_mode) {
        out[vo + k] = proj * wgt;
      } else {
        const double rv = in[vo + k];
        const double loc = rv * wgt;
        const double pv = (loc - proj) * wgt;
        out[vo + k] = pv;
        pc += rv * pv;
        prr += rv * rv;
        ppp += pv * pv;
      }
    }
  }
  double v[3] = {pc, prr, ppp};
  block_sum<3>(v, red);
  if (threadIdx.x == 0 && partials) {
    partials[blockIdx.x * 3 + 0] = v[0];
    partials[blockIdx.x * 3 + 1] = v[1];
    partials[blockIdx.x * 3 + 2] = v[2];
  }
}

// ------------------------------------------------------------------------------------------
// Pass C scalar step: c_next, the trace row, the roundoff floor, every termination test and the
// best-iterate bookkeeping of run_aug (pcg.cpp:157-204), in the reference's order.
__global__ void k_scalar_c(const double* partials, int count, SolveState* st, TraceRowD* rows) {
  if (!st->active) return;
  __shared__ double res[3];
  reduce_partials<3>(partials, count, res);
  if (threadIdx.x != 0) return;
  const double kEps = 2.220446049250313e-16;
  const int64_t i = st->i;
  double c_next = res[0];
  const double rr = res[1], prpr = res[2];
  st->c_next = c_next;
  st->rr = rr;
  st->prpr = prpr;
  st->done = i;
  // w_{i+1} / sw_{i+1} (lambda_i) are materialized into nxt by the next pass A (or k_apply_pending)
  st->upd_pending = 1;
  st->lam_prev = st->lambda;
  st->sampled = (i % st->stride == 0) || c_next <= st->threshold || i == st->max_iter;
  if (i < st->rows_cap) {
    TraceRowD& row = rows[i];
    row.iter = i;
    row.c = c_next;
    row.aug = __longlong_as_double(0x7ff8000000000000LL);
    row.dual = row.aug;
    row.rmse = row.aug;
    row.elapsed_ns = (int64_t)(globaltimer() - st->t0);
  }
  // c_floor (pcg.cpp:81-85)
  const double pr_norm = sqrt(prpr);
  if (rr > 0.0) st->pi_gain = dmax_std(st->pi_gain, pr_norm / sqrt(rr));
  const double floor_c = 16.0 * kEps * dmax_std(st->pi_gain, 1e-3) * rr;
  const double c = st->c;
  const bool exhausted = fabs(c_next) <= floor_c / 64.0 || (fabs(c_next) <= floor_c && c_next <= 1e-6 * c);
  bool stop = false;
  if (c_next < 0.0 && fabs(c_next) > floor_c) {
    st->term = T_BREAKDOWN;
    st->breakdown_iter = i;
    stop = true;
  }
  if (!stop) {
    if (c_next < 0.0) c_next = 0.0;
    if (c_next < st->c_best) {
      st->c_best = c_next;
      st->best = st->nxt;  // where w_{i+1} lands
      st->best_iter = i;
    }
    if (c_next <= st->threshold || exhausted) {
      st->term = T_CONVERGED;
      stop = true;
    }
  }
  if (!stop) {
    if (fabs(c_next - c) <= 1e-15 * c) {
      if (++st->stagnant >= st->stagnation_window) {
        st->term = T_STAGNATION;
        stop = true;
      }
    } else {
      st->stagnant = 0;
    }
  }
  if (!stop && c_next > st->growth_tol * st->c_best && i - st->best_iter >= st->growth_window) {
    st->term = T_BREAKDOWN;
    st->breakdown_iter = i;
    stop = true;
  }
  if (!stop) {
    const double mu = c_next / c;
    st->mu = mu;
    st->c = c_next;
    st->mu_pending = 1;
    if (i == st->max_iter) stop = true;  // loop exhausted: Termination::MaxIter stays
  }
  st->diag_now = (st->diag_every > 0 && (i % st->diag_every) == 0) || stop;
  if (stop) {
    st->active = 0;
    st->cont = 0;
  } else {
    st->cont = 1;
    st->i = i + 1;
  }
}

// Materialize a pending w / sw update after the loop stopped in k_scalar_c (pass A of a next
// iteration never ran): w[nxt] = w[cur] - lambda u, sw[nxt] = sw[cur] - lambda su.
__global__ void k_apply_pending(SolveState* st, WBuf wbuf, const double* u, const double* su, int64_t count) {
  if (!st->upd_pending) return;
  const double lp = st->lam_prev;
  const double *wc = wbuf.w[st->cur], *swc = wbuf.sw[st->cur];
  double *wn = wbuf.w[st->nxt], *swn = wbuf.sw[st->nxt];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    wn[i] = wc[i] + (-lp) * u[i];
    swn[i] = swc[i] + (-lp) * su[i];
  }
}

__global__ void k_finish_pending(SolveState* st) {
  if (!st->upd_pending) return;
  st->cur = st->nxt;
  st->upd_pending = 0;
}

// Trace diagnostics finalize for the row just computed (pcg.cpp:104-116): aug_residual_norm,
// dual_feas_norm, rmse against beta_true when the row is sampled.
__global__ void k_diag_finalize(const double* rpart, int count, const double* xtw, int64_t n, const double* est,
                                const double* beta, SolveState* st, TraceRowD* rows, int64_t row_override) {
  if (row_override < 0 && !st->diag_now) return;
  if (!st->have_beta) beta = nullptr;
  __shared__ double red[32 * 3];
  double v[3] = {0.0, 0.0, 0.0};
  for (int i = threadIdx.x; i < count; i += blockDim.x) v[0] += rpart[i];
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    v[1] += xtw[j] * xtw[j];
    if (beta) {
      const double d = est[j] - beta[j];
      v[2] += d * d;
    }
  }
  block_sum<3>(v, red);
  if (threadIdx.x == 0) {
    const int64_t i = row_override >= 0 ? row_override : st->done;
    if (i < st->rows_cap) {
      TraceRowD& row = rows[i];
      row.aug = sqrt(v[0]);
      row.dual = sqrt(v[1]);
      const bool sampled = row_override >= 0 ? true : (st->sampled != 0);
      if (sampled && beta) row.rmse = sqrt(v[2] / (double)n);
    }
    // the row is final: later (inactive) iterations of the same graph chunk must not redo it (the folded
    // diagnostics' est = R^-1 s_est is computed in place)
    if (row_override < 0) st->diag_now = 0;
  }
}

// ------------------------------------------------------------------------------------------
// Setup QR (SurPreconditioner ctor, structured.cpp:427-450 -> householder_factor / form_q_columns,
// linalg.cpp:24-95) as a TSQR tree per block.  Each work item is one row chunk of one level: the
// leaf factor applies the reference's Householder recipe (alpha = -sign(x_kk) |x|, unit-head v,
// beta = -1/(alpha v0)) to the chunk; the chunk's R goes to the next level, whose QR combines them.
// Q is formed top-down: Q_chunk = H_0 ... H_{n-1} [C; 0] with C the chunk's n x n slice of the
// parent's explicit Q (the identity at the top), as form_q_columns does.
struct QrItem {
  const double* src;   // level matrix (level 0: X_b), column-major ld lds
  int64_t lds;
  int64_t r0, rows;    // chunk rows (of src)
  int64_t rr0;         // first row of the chunk in refl (= r0, or 0 for a tile-contiguous Q tile)
  int64_t rhalf;       // register leaves: offset of row t + 256 from row t in refl (256, or a Q tile)
  int64_t valid;       // rows >= valid of src read as 0 (level 0: M; padding)
  double scale;        // level 0: w_b (DenseMatrix *= w, structured.cpp:435-436); else 1
  double* refl;        // reflector panel / explicit Q destination, ld ldr (same row range)
  int64_t ldr;
  double* tau;         // [n] beta of each reflector
  double* rout;        // R of this chunk: n x n at rout (ld ldo)
  int64_t ldo;
  const double* qpar;  // parent explicit-Q slice (n x n, ld ldp); null = identity
  int64_t ldp;
  double* rdiag;       // top level only: |R_kk| destination for the rank check (else null)
  int n;
  int smem;            // 1: panel in shared memory; 0: in the CTA's global scratch slot
};

constexpr int QR_NT = 256;

__global__ void __launch_bounds__(QR_NT) k_qr_factor(const QrItem* items, int nitems, double* scratch,
                                                     int64_t slot) {
  extern __shared__ double psm[];
  __shared__ double sh[4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = QR_NT / 32;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const QrItem I = items[it];
    const int n = I.n;
    const int64_t L = I.rows;
    double* P = I.smem ? psm : scratch + (int64_t)blockIdx.x * slot;
    __syncthreads();
    for (int64_t idx = threadIdx.x; idx < L * n; idx += QR_NT) {
      const int j = (int)(idx / L);
      const int64_t i = idx - (int64_t)j * L;
      const int64_t row = I.r0 + i;
      P[idx] = (row < I.valid) ? I.src[(int64_t)j * I.lds + row] * I.scale : 0.0;
    }
    __syncthreads();
    for (int k = 0; k < n; ++k) {
      double* Pk = P + (int64_t)k * L;
      if (warp == 0) {
        double amax = 0.0;
        for (int64_t i = k + lane; i < L; i += 32) amax = fmax(amax, fabs(Pk[i]));
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) amax = fmax(amax, __shfl_xor_sync(FULL, amax, o));
        double ssq = 0.0;
        if (amax > 0.0)
          for (int64_t i = k + lane; i < L; i += 32) {
            const double t = Pk[i] / amax;
            ssq += t * t;
          }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) ssq += __shfl_xor_sync(FULL, ssq, o);
        const double norm_x = amax * sqrt(ssq);
        double alpha = 0.0, v0 = 1.0, beta = 0.0;
        if (norm_x != 0.0) {
          const double wkk = Pk[k];
          alpha = wkk >= 0.0 ? -norm_x : norm_x;
          v0 = wkk - alpha;
          beta = -1.0 / (alpha * v0);
        }
        __syncwarp();
        if (norm_x != 0.0) {
          for (int64_t i = k + 1 + lane; i < L; i += 32) Pk[i] /= v0;
          if (lane == 0) Pk[k] = v0;
        }
        if (lane == 0) {
          sh[0] = alpha;
          sh[1] = v0;
          sh[2] = beta;
          I.tau[k] = beta;
        }
      }
      __syncthreads();
      const double beta = sh[2];
      if (beta != 0.0) {
        const double v0 = sh[1];
        const double beta_hat = beta * v0 * v0;
        for (int j = k + 1 + warp; j < n; j += NW) {
          double* Pj = P + (int64_t)j * L;
          double s = 0.0;
          for (int64_t i = k + 1 + lane; i < L; i += 32) s += Pk[i] * Pj[i];
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
          s = (Pj[k] + s) * beta_hat;
          __syncwarp();
          if (lane == 0) Pj[k] -= s;
          for (int64_t i = k + 1 + lane; i < L; i += 32) Pj[i] -= s * Pk[i];
        }
      }
      if (threadIdx.x == 0) {
        // r_diag[k] = alpha: keep it beside the packed panel (R output below)
        sh[3] = sh[0];
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        I.rout[k + (int64_t)k * I.ldo] = sh[3];
        if (I.rdiag) I.rdiag[k] = sh[3];
      }
    }
    __syncthreads();
    // R (strict upper part from the panel; diagonal written above; zeros below)
    for (int idx = threadIdx.x; idx < n * n; idx += QR_NT) {
      const int j = idx / n, i = idx - j * n;
      if (i < j) I.rout[i + (int64_t)j * I.ldo] = P[i + (int64_t)j * L];
      else if (i > j) I.rout[i + (int64_t)j * I.ldo] = 0.0;
    }
    // packed reflectors to the level storage
    for (int64_t idx = threadIdx.x; idx < L * n; idx += QR_NT) {
      const int j = (int)(idx / L);
      const int64_t i = idx - (int64_t)j * L;
      I.refl[(int64_t)j * I.ldr + I.rr0 + i] = P[idx];
    }
  }
}

// Explicit thin Q of a chunk: E = H_0 ... H_{n-1} [C; 0], warp per column, the column held in
// registers (NQ x 32 rows); reflectors read from the staged panel.
template <int NQ>
__global__ void __launch_bounds__(QR_NT) k_qr_formq(const QrItem* items, int nitems, double* scratch, int64_t slot) {
  extern __shared__ double psm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = QR_NT / 32;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const QrItem I = items[it];
    const int n = I.n;
    const int64_t L = I.rows;
    double* P = I.smem ? psm : scratch + (int64_t)blockIdx.x * slot;
    __syncthreads();
    for (int64_t idx = threadIdx.x; idx < L * n; idx += QR_NT) {
      const int j = (int)(idx / L);
      const int64_t i = idx - (int64_t)j * L;
      P[idx] = I.refl[(int64_t)j * I.ldr + I.rr0 + i];
    }
    __syncthreads();
    for (int j = warp; j < n; j += NW) {
      double e[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int64_t i = lane + 32 * q;
        double v = 0.0;
        if (i < n) v = I.qpar ? I.qpar[i + (int64_t)j * I.ldp] : (i == j ? 1.0 : 0.0);
        e[q] = v;
      }
      for (int k = n - 1; k >= 0; --k) {
        const double beta = I.tau[k];
        if (beta == 0.0) continue;
        const double* Pk = P + (int64_t)k * L;
        const double v0 = Pk[k];
        const double beta_hat = beta * v0 * v0;
        // s = e[k] + sum_{i>k} P[i,k] e[i]
        double s = 0.0, ek = 0.0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int64_t i = lane + 32 * q;
          if (i > k && i < L) s += Pk[i] * e[q];
          if (i == k) ek = e[q];
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
        ek = __shfl_sync(FULL, ek, k & 31);
        s = (ek + s) * beta_hat;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int64_t i = lane + 32 * q;
          if (i == k) e[q] -= s;
          else if (i > k && i < L) e[q] -= s * Pk[i];
        }
      }
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int64_t i = lane + 32 * q;
        if (i < L) I.refl[(int64_t)j * I.ldr + I.rr0 + i] = e[q];
      }
    }
  }
}

// ------------------------------------------------------------------------------------------
// Register-resident TSQR leaves for narrow blocks (n <= 32, chunk rows <= RPT * 256): thread t owns
// rows t + 256 h (h < RPT) of the chunk in registers.  Per Householder step one block reduction of 32
// values (the column norm and every trailing dot at once); the k loop stays rolled (the factor rotates
// its rows left one column per step) so the code stays in the instruction cache.
constexpr int QRR_NT = 256;
constexpr int QRR_RPT = 2;                 // rows per thread
constexpr int QRR_ROWS = QRR_NT * QRR_RPT;  // leaf rows

// acc[j] summed over the CTA (fixed order) -> out[j] (shared), all threads see it after the call
template <int NB>
__device__ __forceinline__ void block_vec_sum(double (&acc)[NB], double (*red)[NB], double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  warp_transpose_reduce<NB>(acc);
  red[warp][lane % NB] = acc[0];
  __syncthreads();
  if (threadIdx.x < NB) {
    double s = 0.0;
    for (int w = 0; w < QRR_NT / 32; ++w) s += red[w][threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

// row (t + 256 h) of a chunk in the reflector / Q storage: column-major (ld ldr) or, for a level-0
// leaf of tile-contiguous Q, two 256-row tiles rhalf doubles apart
__device__ __forceinline__ int64_t qr_row_off(const QrItem& I, int j, int t, int h) {
  return (int64_t)j * I.ldr + I.rr0 + t + (int64_t)h * I.rhalf;
}

template <int NB>
__global__ void __launch_bounds__(QRR_NT, 1) k_qr_factor_reg(const QrItem* items, int nitems) {
  __shared__ double red_v[QRR_NT / 32][NB];
  __shared__ double svec[NB];
  __shared__ double rowk[2][NB];
  __shared__ double redm[QRR_NT / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const QrItem I = items[it];
    const int n = I.n;
    const int64_t L = I.rows;
    double a[QRR_RPT][NB];
#pragma unroll
    for (int h = 0; h < QRR_RPT; ++h) {
      const int64_t rl = t + h * QRR_NT;
      const int64_t row = I.r0 + rl;
#pragma unroll
      for (int j = 0; j < NB; ++j)
        a[h][j] = (rl < L && j < n && row < I.valid) ? I.src[(int64_t)j * I.lds + row] * I.scale : 0.0;
    }
    // exact power-of-two pre-scale of the leaf so the plain sums of squares below cannot overflow
    double mx = 0.0;
#pragma unroll
    for (int h = 0; h < QRR_RPT; ++h)
#pragma unroll
      for (int j = 0; j < NB; ++j) mx = fmax(mx, fabs(a[h][j]));
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
    if (lane == 0) redm[warp] = mx;
    __syncthreads();
    mx = redm[0];
    for (int w = 1; w < QRR_NT / 32; ++w) mx = fmax(mx, redm[w]);
    int ex = 0;
    if (mx > 0.0) frexp(mx, &ex);
    const double sc = ldexp(1.0, -ex), unsc = ldexp(1.0, ex);
#pragma unroll
    for (int h = 0; h < QRR_RPT; ++h)
#pragma unroll
      for (int j = 0; j < NB; ++j) a[h][j] *= sc;
    // Row rotation: at step k, a[h][0] is column k and a[h][j] column k + j.
#pragma unroll 1
    for (int k = 0; k < n; ++k) {
      const int ntr = n - k;
      // one reduction per column: S_0 = x'x (x = column k, rows >= k) and S_j = x'a_{k+j}
      double x[QRR_RPT];
#pragma unroll
      for (int h = 0; h < QRR_RPT; ++h) x[h] = (t + h * QRR_NT >= k) ? a[h][0] : 0.0;
      if (t == (k & (QRR_NT - 1))) {  // the owner of row k (h = k / 256)
        const int hk = k / QRR_NT;
#pragma unroll
        for (int h = 0; h < QRR_RPT; ++h)
          if (h == hk)
#pragma unroll
            for (int j = 0; j < NB; ++j) rowk[k & 1][j] = a[h][j];
      }
      double acc[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        double s = 0.0;
#pragma unroll
        for (int h = 0; h < QRR_RPT; ++h) s += x[h] * a[h][j];
        acc[j] = (j < ntr) ? s : 0.0;
      }
      block_vec_sum<NB>(acc, red_v, svec);  // two __syncthreads
      const double norm_x = sqrt(svec[0]);
      const double wkk = rowk[k & 1][0];
      double beta = 0.0, v0 = 1.0, alpha = 0.0;
      if (norm_x != 0.0) {
        alpha = wkk >= 0.0 ? -norm_x : norm_x;
        v0 = wkk - alpha;
        beta = -1.0 / (alpha * v0);
      }
      if (t == 0) I.tau[k] = beta;
      const double inv_v0 = 1.0 / v0, inv_alpha = (alpha != 0.0) ? 1.0 / alpha : 0.0;
      // update factor s_j beta_hat = -(x'a_j - alpha a_kj) / alpha   (beta_hat = -v0 / alpha)
#pragma unroll
      for (int h = 0; h < QRR_RPT; ++h) {
        const int rl = t + h * QRR_NT;
        double v = 0.0;       // this row's reflector component (unit head)
        double col = a[h][0]; // final packed-panel entry of column k for this row
        if (norm_x != 0.0) {
          if (rl > k) {
            col = a[h][0] * inv_v0;
            v = col;
          } else if (rl == k) {
            v = 1.0;
            col = v0;
          }
#pragma unroll
          for (int j = 1; j < NB; ++j)
            if (j < ntr) a[h][j] -= ((alpha * rowk[k & 1][j] - svec[j]) * inv_alpha) * v;
        }
        if (rl < L) I.refl[qr_row_off(I, k, t, h)] = col;
        if (rl < n) {  // R column k: R(rl, k) for rl < k, alpha on the diagonal, zero below
          const double r = (rl < k) ? a[h][0] : (rl == k ? alpha : 0.0);
          I.rout[rl + (int64_t)k * I.ldo] = r * unsc;
        }
        // rotate the row left by one column
#pragma unroll
        for (int j = 0; j < NB - 1; ++j) a[h][j] = a[h][j + 1];
        a[h][NB - 1] = 0.0;
      }
    }
    __syncthreads();
  }
}

// Explicit thin Q of a narrow chunk: E = H_0 ... H_{n-1} [C; 0]; the output rows in registers, the
// packed reflectors staged in shared memory (rows x n, <= 128 KB).
template <int NB>
__global__ void __launch_bounds__(QRR_NT, 1) k_qr_formq_reg(const QrItem* items, int nitems) {
  extern __shared__ double P[];  // [NB][QRR_ROWS]
  __shared__ double red_v[QRR_NT / 32][NB];
  __shared__ double svec[NB];
  const int t = threadIdx.x;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const QrItem I = items[it];
    const int n = I.n;
    const int64_t L = I.rows;
    __syncthreads();
    for (int j = 0; j < n; ++j)
#pragma unroll
      for (int h = 0; h < QRR_RPT; ++h) {
        const int rl = t + h * QRR_NT;
        P[j * QRR_ROWS + rl] = (rl < L) ? I.refl[qr_row_off(I, j, t, h)] : 0.0;
      }
    double e[QRR_RPT][NB];
#pragma unroll
    for (int h = 0; h < QRR_RPT; ++h)
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int rl = t + h * QRR_NT;
        double v = 0.0;
        if (rl < n && j < n) v = I.qpar ? I.qpar[rl + (int64_t)j * I.ldp] : (rl == j ? 1.0 : 0.0);
        e[h][j] = v;
      }
    __syncthreads();
#pragma unroll 1
    for (int k = n - 1; k >= 0; --k) {
      const double beta = I.tau[k];
      if (beta == 0.0) continue;  // form_q_columns skips zero reflectors (linalg.cpp:83)
      const double v0 = P[k * QRR_ROWS + k];
      const double beta_hat = beta * v0 * v0;
      double v[QRR_RPT];
#pragma unroll
      for (int h = 0; h < QRR_RPT; ++h) {
        const int rl = t + h * QRR_NT;
        v[h] = (rl > k && rl < L) ? P[k * QRR_ROWS + rl] : (rl == k ? 1.0 : 0.0);
      }
      double acc[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        double s = 0.0;
#pragma unroll
        for (int h = 0; h < QRR_RPT; ++h) s += v[h] * e[h][j];
        acc[j] = s;
      }
      block_vec_sum<NB>(acc, red_v, svec);
#pragma unroll
      for (int h = 0; h < QRR_RPT; ++h)
#pragma unroll
        for (int j = 0; j < NB; ++j) e[h][j] -= (svec[j] * beta_hat) * v[h];
    }
#pragma unroll
    for (int h = 0; h < QRR_RPT; ++h) {
      const int rl = t + h * QRR_NT;
#pragma unroll
      for (int j = 0; j < NB; ++j)
        if (j < n && rl < L) I.refl[qr_row_off(I, j, t, h)] = e[h][j];
    }
  }
}

// ------------------------------------------------------------------------------------------
// Lane-per-column TSQR leaves (n <= 32, chunk rows <= 256).  Lane j of every warp owns column j; the
// chunk's rows are interleaved across the 8 warps (warp w, slot i: row 8 i + w), so the top 32 rows
// -- the only ones that need step-dependent masking -- are spread 4 per warp and every warp does the
// same work.  Per Householder step k (the reference recipe, linalg.cpp:24-63: alpha = -sign(x_kk) |x|,
// unit-head v, beta = -1 / (alpha v0)):
//   * x = column k, broadcast from lane k with shuffles (rows < k masked to 0);
//   * S_j = x . a_j for every column at once: per-lane dot over the warp's rows, then one CTA reduction
//     (one barrier per step, double-buffered); row k comes with it;
//   * a_j -= f_j v, f_j = (alpha a_kj - S_j) / alpha, v = x / v0 (unit head): one FMA per entry.
// Panels move global <-> shared with coalesced row-per-thread accesses; the next chunk's panel is
// prefetched (cp.async, zero-filled padding) while the current one is factored.  Not bitwise the
// reference's sequential Householder (the TSQR tree reorders it anyway): FMA is used explicitly.
constexpr int QRC_NT = 256;
constexpr int QRC_ROWS = 256;                 // leaf rows (one 256-row Q tile)
constexpr int QRC_LD = QRC_ROWS + 1;          // panel column stride in shared memory (odd)
constexpr int QRC_PANEL = 32 * QRC_LD;        // doubles per panel buffer
constexpr size_t qrc_smem_bytes() { return (size_t)2 * QRC_PANEL * sizeof(double); }

__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }

__device__ __forceinline__ void cp_async8_zfill(double* dst, const double* src, bool valid) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  const int bytes = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(valid ? src : nullptr), "r"(bytes)
               : "memory");
}

// row t (= threadIdx.x) of a leaf panel into P (columns j < 32; zero past n, past the chunk, past valid)
__device__ __forceinline__ void qrc_prefetch(double* P, const double* src, int64_t lds, int64_t r0, int64_t rows,
                                             int64_t valid, int n) {
  const int t = threadIdx.x;
  const bool rv = t < rows && r0 + t < valid;
  for (int j = 0; j < 32; ++j) cp_async8_zfill(P + j * QRC_LD + t, src + (int64_t)j * lds + r0 + t, rv && j < n);
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__global__ void __launch_bounds__(QRC_NT, 1) k_qr_factor_lc(const QrItem* items, int nitems) {
  extern __shared__ double SB[];                // 2 panel buffers [32][QRC_LD]
  __shared__ double red[2][QRC_NT / 32][32];
  __shared__ double rowk[2][32];
  __shared__ double alph[32];
  __shared__ double redm[QRC_NT / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int buf = 0;
  if (blockIdx.x < nitems) {
    const QrItem I0 = items[blockIdx.x];
    qrc_prefetch(SB, I0.src, I0.lds, I0.r0, I0.rows, I0.valid, I0.n);
  }
  for (int it = blockIdx.x; it < nitems; it += gridDim.x, buf ^= 1) {
    const QrItem I = items[it];
    const int n = I.n;
    const int64_t L = I.rows;
    double* S = SB + buf * QRC_PANEL;
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();                            // panel landed; the other buffer's readers are done
    if (it + (int)gridDim.x < nitems) {
      const QrItem& In = items[it + gridDim.x];
      qrc_prefetch(SB + (buf ^ 1) * QRC_PANEL, In.src, In.lds, In.r0, In.rows, In.valid, In.n);
    }
    double* col = S + lane * QRC_LD;            // this lane's column
    double a[32];
    double mx = 0.0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      a[i] = col[8 * i + warp] * I.scale;
      mx = fmax(mx, fabs(a[i]));
    }
    // exact power-of-two pre-scale so the plain sums of squares cannot overflow
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
    if (lane == 0) redm[warp] = mx;
    __syncthreads();
    mx = redm[0];
#pragma unroll
    for (int w = 1; w < QRC_NT / 32; ++w) mx = fmax(mx, redm[w]);
    int ex = 0;
    if (mx > 0.0) frexp(mx, &ex);
    const double sc = ldexp(1.0, -ex), unsc = ldexp(1.0, ex);
#pragma unroll
    for (int i = 0; i < 32; ++i) a[i] *= sc;
    double my_inv = 1.0, my_v0 = 0.0;           // this lane's own reflector (step k == lane)
#pragma unroll 1
    for (int k = 0; k < n; ++k) {
      const int par = k & 1;
      double x[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) x[i] = __shfl_sync(FULL, a[i], k);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (8 * i + warp < k) x[i] = 0.0;       // rows above k are R rows
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        s0 = fma_rn(x[i + 0], a[i + 0], s0);
        s1 = fma_rn(x[i + 1], a[i + 1], s1);
        s2 = fma_rn(x[i + 2], a[i + 2], s2);
        s3 = fma_rn(x[i + 3], a[i + 3], s3);
      }
      if (warp == (k & 7)) {                    // row k = slot k / 8 of warp k % 8
        const int sk = k >> 3;
        rowk[par][lane] = sk == 0 ? a[0] : sk == 1 ? a[1] : sk == 2 ? a[2] : a[3];
      }
      red[par][warp][lane] = (s0 + s1) + (s2 + s3);
      __syncthreads();
      double sj = 0.0;
#pragma unroll
      for (int w = 0; w < QRC_NT / 32; ++w) sj += red[par][w][lane];
      const double skk = __shfl_sync(FULL, sj, k);
      const double akj = rowk[par][lane];
      const double wkk = rowk[par][k];
      const double norm_x = sqrt(skk);
      double alpha = 0.0, v0 = 1.0, beta = 0.0, inv_alpha = 0.0, inv_v0 = 1.0;
      if (norm_x != 0.0) {
        alpha = wkk >= 0.0 ? -norm_x : norm_x;
        v0 = wkk - alpha;
        const double dd = 1.0 / (alpha * v0);
        beta = -dd;
        inv_alpha = v0 * dd;
        inv_v0 = alpha * dd;
      }
      const double f = (lane > k && lane < n) ? (alpha * akj - sj) * inv_alpha : 0.0;
      const double g = f * inv_v0;
      if (lane == k) {
        my_inv = inv_v0;
        my_v0 = (norm_x != 0.0) ? v0 : wkk;
      }
      if (t == k) {
        alph[k] = alpha;
        I.tau[k] = beta;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double up = fma_rn(-g, x[i], a[i]);
        a[i] = (8 * i + warp == k) ? a[i] - f : up;
      }
#pragma unroll
      for (int i = 4; i < 32; ++i) a[i] = fma_rn(-g, x[i], a[i]);
    }
    // packed reflector panel: rows > j of column j scaled by 1 / v0_j, v0_j on the diagonal, R above
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int r = 8 * i + warp;
      double v = a[i];
      if (i >= 4 || r > lane) v = a[i] * my_inv;
      else if (r == lane) v = my_v0;
      col[r] = v;
    }
    __syncthreads();
    // R (scaled back), the diagonal from alpha; zeros below
    for (int idx = t; idx < n * n; idx += QRC_NT) {
      const int j = idx / n, i = idx - j * n;
      const double r = (i < j) ? S[j * QRC_LD + i] * unsc : (i == j ? alph[j] * unsc : 0.0);
      I.rout[i + (int64_t)j * I.ldo] = r;
      if (i == j && I.rdiag) I.rdiag[j] = r;
    }
    // reflector panel out (coalesced: thread per row)
    if (t < L)
      for (int j = 0; j < n; ++j) I.refl[(int64_t)j * I.ldr + I.rr0 + t] = S[j * QRC_LD + t];
  }
}

// Explicit thin Q of a narrow chunk: E = H_0 ... H_{n-1} [C; 0] (form_q_columns, linalg.cpp:65-95),
// lane j = column j of E, rows interleaved across warps in registers; the packed reflectors staged in
// shared memory, their top 32 rows pre-masked (unit head, zeros above: V0) so every read is a plain
// broadcast.  The next chunk's panel is prefetched while the current one is formed.
__global__ void __launch_bounds__(QRC_NT, 1) k_qr_formq_lc(const QrItem* items, int nitems) {
  extern __shared__ double SB[];                // 2 packed-panel buffers [32][QRC_LD]
  __shared__ double V0[32][33];                 // masked reflector columns, rows 0..31
  __shared__ double bh[32];                     // beta_hat = beta v0^2 per reflector
  __shared__ int tz[32];                        // reflector k is zero (beta == 0)
  __shared__ double red[2][QRC_NT / 32][32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int buf = 0;
  if (blockIdx.x < nitems) {
    const QrItem I0 = items[blockIdx.x];
    qrc_prefetch(SB, I0.refl + I0.rr0, I0.ldr, 0, I0.rows, I0.rows, I0.n);
  }
  for (int it = blockIdx.x; it < nitems; it += gridDim.x, buf ^= 1) {
    const QrItem I = items[it];
    const int n = I.n;
    const int64_t L = I.rows;
    double* S = SB + buf * QRC_PANEL;
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    if (it + (int)gridDim.x < nitems) {
      const QrItem& In = items[it + gridDim.x];
      qrc_prefetch(SB + (buf ^ 1) * QRC_PANEL, In.refl + In.rr0, In.ldr, 0, In.rows, In.rows, In.n);
    }
    for (int idx = t; idx < 32 * 32; idx += QRC_NT) {
      const int k = idx >> 5, i = idx & 31;
      const double pk = S[k * QRC_LD + i];
      V0[k][i] = (i > k && i < L) ? pk : (i == k ? 1.0 : 0.0);
      if (i == k) {
        const double tk = (k < n) ? I.tau[k] : 0.0;
        bh[k] = tk * pk * pk;
        tz[k] = (tk == 0.0);
      }
    }
    double e[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int r = 8 * i + warp;
      double v = 0.0;
      if (i < 4 && r < n && lane < n) v = I.qpar ? I.qpar[r + (int64_t)lane * I.ldp] : (r == lane ? 1.0 : 0.0);
      e[i] = v;
    }
    __syncthreads();
#pragma unroll 1
    for (int k = n - 1; k >= 0; --k) {
      if (tz[k]) continue;  // form_q_columns skips zero reflectors (linalg.cpp:83)
      const double bhk = bh[k];
      const int par = k & 1;
      double v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = (i < 4) ? V0[k][8 * i + warp] : S[k * QRC_LD + 8 * i + warp];
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        s0 = fma_rn(v[i + 0], e[i + 0], s0);
        s1 = fma_rn(v[i + 1], e[i + 1], s1);
        s2 = fma_rn(v[i + 2], e[i + 2], s2);
        s3 = fma_rn(v[i + 3], e[i + 3], s3);
      }
      red[par][warp][lane] = (s0 + s1) + (s2 + s3);
      __syncthreads();
      double sj = 0.0;
#pragma unroll
      for (int w = 0; w < QRC_NT / 32; ++w) sj += red[par][w][lane];
      const double h = -(sj * bhk);
#pragma unroll
      for (int i = 0; i < 32; ++i) e[i] = fma_rn(h, v[i], e[i]);
    }
    // E out through the panel (coalesced)
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 32; ++i) S[lane * QRC_LD + 8 * i + warp] = e[i];
    __syncthreads();
    if (t < L)
      for (int j = 0; j < n; ++j) I.refl[(int64_t)j * I.ldr + I.rr0 + t] = S[j * QRC_LD + t];
  }
}

// ------------------------------------------------------------------------------------------
// Two-CTA-per-SM forms of the lane-per-column leaves (the default).  The leaf kernels above are bound by the
// latency of their 32 dependent steps (one CTA reduction + a sqrt and a divide per step) with one CTA per SM;
// these keep no broadcast copy of column k in registers (it is re-read from lane k with shuffles in the update)
// and stage one panel instead of two, so two CTAs -- two independent leaves -- share each SM and hide each
// other's step latency.  Same arithmetic, operation for operation, as k_qr_factor_lc / k_qr_formq_lc.
constexpr size_t qrc2_smem_bytes() { return (size_t)QRC_PANEL * sizeof(double); }

__global__ void __launch_bounds__(QRC_NT, 2) k_qr_factor_lc2(const QrItem* items, int nitems) {
  extern __shared__ double S[];                 // one panel buffer [32][QRC_LD]
  __shared__ double red[2][QRC_NT / 32][32];
  __shared__ double rowk[2][32];
  __shared__ double alph[32];
  __shared__ double redm[QRC_NT / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const QrItem I = items[it];
    const int n = I.n;
    const int64_t L = I.rows;
    __syncthreads();                            // the previous item's panel readers are done
    qrc_prefetch(S, I.src, I.lds, I.r0, I.rows, I.valid, I.n);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    double* col = S + lane * QRC_LD;            // this lane's column
    double a[32];
    double mx = 0.0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      a[i] = col[8 * i + warp] * I.scale;
      mx = fmax(mx, fabs(a[i]));
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
    if (lane == 0) redm[warp] = mx;
    __syncthreads();
    mx = redm[0];
#pragma unroll
    for (int w = 1; w < QRC_NT / 32; ++w) mx = fmax(mx, redm[w]);
    int ex = 0;
    if (mx > 0.0) frexp(mx, &ex);
    const double sc = ldexp(1.0, -ex), unsc = ldexp(1.0, ex);
#pragma unroll
    for (int i = 0; i < 32; ++i) a[i] *= sc;
    double my_inv = 1.0, my_v0 = 0.0;
#pragma unroll 1
    for (int k = 0; k < n; ++k) {
      const int par = k & 1;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        double x0 = __shfl_sync(FULL, a[i + 0], k), x1 = __shfl_sync(FULL, a[i + 1], k);
        double x2 = __shfl_sync(FULL, a[i + 2], k), x3 = __shfl_sync(FULL, a[i + 3], k);
        if (i == 0) {
          if (0 * 8 + warp < k) x0 = 0.0;
          if (1 * 8 + warp < k) x1 = 0.0;
          if (2 * 8 + warp < k) x2 = 0.0;
          if (3 * 8 + warp < k) x3 = 0.0;
        }
        s0 = fma_rn(x0, a[i + 0], s0);
        s1 = fma_rn(x1, a[i + 1], s1);
        s2 = fma_rn(x2, a[i + 2], s2);
        s3 = fma_rn(x3, a[i + 3], s3);
      }
      if (warp == (k & 7)) {
        const int sk = k >> 3;
        rowk[par][lane] = sk == 0 ? a[0] : sk == 1 ? a[1] : sk == 2 ? a[2] : a[3];
      }
      red[par][warp][lane] = (s0 + s1) + (s2 + s3);
      __syncthreads();
      double sj = 0.0;
#pragma unroll
      for (int w = 0; w < QRC_NT / 32; ++w) sj += red[par][w][lane];
      const double skk = __shfl_sync(FULL, sj, k);
      const double akj = rowk[par][lane];
      const double wkk = rowk[par][k];
      const double norm_x = sqrt(skk);
      double alpha = 0.0, v0 = 1.0, beta = 0.0, inv_alpha = 0.0, inv_v0 = 1.0;
      if (norm_x != 0.0) {
        alpha = wkk >= 0.0 ? -norm_x : norm_x;
        v0 = wkk - alpha;
        const double dd = 1.0 / (alpha * v0);
        beta = -dd;
        inv_alpha = v0 * dd;
        inv_v0 = alpha * dd;
      }
      const double f = (lane > k && lane < n) ? (alpha * akj - sj) * inv_alpha : 0.0;
      const double gg = f * inv_v0;
      if (lane == k) {
        my_inv = inv_v0;
        my_v0 = (norm_x != 0.0) ? v0 : wkk;
      }
      if (t == k) {
        alph[k] = alpha;
        I.tau[k] = beta;
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        double x = __shfl_sync(FULL, a[i], k);  // lane k's column is unchanged by its own step (f = 0 there)
        if (i < 4 && 8 * i + warp < k) x = 0.0;
        const double up = fma_rn(-gg, x, a[i]);
        a[i] = (i < 4 && 8 * i + warp == k) ? a[i] - f : up;
      }
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int r = 8 * i + warp;
      double v = a[i];
      if (i >= 4 || r > lane) v = a[i] * my_inv;
      else if (r == lane) v = my_v0;
      col[r] = v;
    }
    __syncthreads();
    for (int idx = t; idx < n * n; idx += QRC_NT) {
      const int j = idx / n, i = idx - j * n;
      const double r = (i < j) ? S[j * QRC_LD + i] * unsc : (i == j ? alph[j] * unsc : 0.0);
      I.rout[i + (int64_t)j * I.ldo] = r;
      if (i == j && I.rdiag) I.rdiag[j] = r;
    }
    if (t < L)
      for (int j = 0; j < n; ++j) I.refl[(int64_t)j * I.ldr + I.rr0 + t] = S[j * QRC_LD + t];
  }
}

__global__ void __launch_bounds__(QRC_NT, 2) k_qr_formq_lc2(const QrItem* items, int nitems) {
  extern __shared__ double S[];                 // one packed-panel buffer [32][QRC_LD]
  __shared__ double V0[32][33];
  __shared__ double bh[32];
  __shared__ int tz[32];
  __shared__ double red[2][QRC_NT / 32][32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const QrItem I = items[it];
    const int n = I.n;
    const int64_t L = I.rows;
    __syncthreads();
    qrc_prefetch(S, I.refl + I.rr0, I.ldr, 0, I.rows, I.rows, I.n);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    for (int idx = t; idx < 32 * 32; idx += QRC_NT) {
      const int k = idx >> 5, i = idx & 31;
      const double pk = S[k * QRC_LD + i];
      V0[k][i] = (i > k && i < L) ? pk : (i == k ? 1.0 : 0.0);
      if (i == k) {
        const double tk = (k < n) ? I.tau[k] : 0.0;
        bh[k] = tk * pk * pk;
        tz[k] = (tk == 0.0);
      }
    }
    double e[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int r = 8 * i + warp;
      double v = 0.0;
      if (i < 4 && r < n && lane < n) v = I.qpar ? I.qpar[r + (int64_t)lane * I.ldp] : (r == lane ? 1.0 : 0.0);
      e[i] = v;
    }
    __syncthreads();
#pragma unroll 1
    for (int k = n - 1; k >= 0; --k) {
      if (tz[k]) continue;
      const double bhk = bh[k];
      const int par = k & 1;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        const double v0_ = (i < 4) ? V0[k][8 * (i + 0) + warp] : S[k * QRC_LD + 8 * (i + 0) + warp];
        const double v1_ = (i < 4) ? V0[k][8 * (i + 1) + warp] : S[k * QRC_LD + 8 * (i + 1) + warp];
        const double v2_ = (i < 4) ? V0[k][8 * (i + 2) + warp] : S[k * QRC_LD + 8 * (i + 2) + warp];
        const double v3_ = (i < 4) ? V0[k][8 * (i + 3) + warp] : S[k * QRC_LD + 8 * (i + 3) + warp];
        s0 = fma_rn(v0_, e[i + 0], s0);
        s1 = fma_rn(v1_, e[i + 1], s1);
        s2 = fma_rn(v2_, e[i + 2], s2);
        s3 = fma_rn(v3_, e[i + 3], s3);
      }
      red[par][warp][lane] = (s0 + s1) + (s2 + s3);
      __syncthreads();
      double sj = 0.0;
#pragma unroll
      for (int w = 0; w < QRC_NT / 32; ++w) sj += red[par][w][lane];
      const double h = -(sj * bhk);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const double v = (i < 4) ? V0[k][8 * i + warp] : S[k * QRC_LD + 8 * i + warp];
        e[i] = fma_rn(h, v, e[i]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 32; ++i) S[lane * QRC_LD + 8 * i + warp] = e[i];
    __syncthreads();
    if (t < L)
      for (int j = 0; j < n; ++j) I.refl[(int64_t)j * I.ldr + I.rr0 + t] = S[j * QRC_LD + t];
  }
}

// ------------------------------------------------------------------------------------------
// Explicit Q of a narrow leaf in compact WY form on the FP64 tensor cores (round 2, the default).  The leaf's n
// reflectors H_j = I - bh_j v_j v_j' (unit-head v_j, bh_j = beta_j v0_j^2: the reference's recipe) multiply to
// H_0 ... H_{n-1} = I - V T V' with T upper triangular, T_jj = bh_j, T_{0:j,j} = -bh_j T_{0:j,0:j} (V'V)_{0:j,j}
// (the forward accumulation of form_q_columns' product, linalg.cpp:77-95, as LAPACK's larft does).  So
// E = H_0 ... H_{n-1} [C; 0] = [C; 0] - V (T (V_top' C)), with V'V and the final V (T ...) product as DMMA
// m16n8k4 tiles: one read of the packed panel, one write of E, and no per-reflector CTA reductions (the
// lane-per-column k_qr_formq_lc2 runs 32 dependent reduction steps per leaf).  Rounding differs from applying the
// reflectors one by one only in the order of the sums (Q stays orthonormal to ~1e-15; the TSQR tests pin it).
constexpr int QW_NT = 256;
constexpr int QW_LDV = 256 + 4;  // V column stride in shared memory (conflict-free DMMA fragment loads)
constexpr int QW_LDS = 33;       // 32 x 32 scratch matrices
constexpr size_t qw_smem_bytes() { return (size_t)(32 * QW_LDV + 6 * 32 * QW_LDS) * sizeof(double); }

__global__ void __launch_bounds__(QW_NT, 2) k_qr_formq_wy(const QrItem* items, int nitems) {
  extern __shared__ double sm[];
  double* Vs = sm;                           // V, column j at Vs + j QW_LDV (rows 0..255)
  double* Gp = Vs + 32 * QW_LDV;             // two K-half partials of V'V, [2][32][QW_LDS]
  double* Ts = Gp + 2 * 32 * QW_LDS;         // T
  double* Ys = Ts + 32 * QW_LDS;             // V_top' C, then -(T Y)
  double* Zs = Ys + 32 * QW_LDS;
  double* Cs = Zs + 32 * QW_LDS;             // the parent's n x n slice C (or I)
  __shared__ double bh[32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int g = lane >> 2, q4 = lane & 3;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const QrItem I = items[it];
    const int n = I.n;
    const int64_t L = I.rows;
    __syncthreads();  // the previous item's readers of shared memory are done
    {
      const bool rv = t < L;
      for (int j = 0; j < 32; ++j)
        cp_async8_zfill(Vs + j * QW_LDV + t, I.refl + I.rr0 + (int64_t)j * I.ldr + t, rv && j < n);
      for (int idx = t; idx < 32 * 32; idx += QW_NT) {  // C row-major in Cs[r][c]
        const int c = idx >> 5, r = idx & 31;
        if (I.qpar) cp_async8_zfill(Cs + r * QW_LDS + c, I.qpar + r + (int64_t)c * I.ldp, r < n && c < n);
        else Cs[r * QW_LDS + c] = (r == c && r < n) ? 1.0 : 0.0;
      }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    if (t < 32) {  // bh_j = beta_j v0_j^2 from the packed diagonal, before the unit head replaces it
      const double v0 = Vs[t * QW_LDV + t];
      const double tk = (t < n) ? I.tau[t] : 0.0;
      bh[t] = tk * v0 * v0;
    }
    __syncthreads();
    for (int idx = t; idx < 32 * 32; idx += QW_NT) {  // unit head, zeros above (the R part of the packed panel)
      const int j = idx >> 5, r = idx & 31;
      if (r < j) Vs[j * QW_LDV + r] = 0.0;
      else if (r == j) Vs[j * QW_LDV + r] = (j < n && bh[j] != 0.0) ? 1.0 : 0.0;
    }
    __syncthreads();
    // V'V: warp w -> Gram columns [8 (w & 3), +8), rows [128 (w >> 2), +128) of V
    {
      double acc[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
      const int c0 = 8 * (warp & 3), rb = 128 * (warp >> 2);
#pragma unroll 4
      for (int kk = 0; kk < 32; ++kk) {
        const int r0 = rb + 4 * kk;
        const double b0 = Vs[(c0 + g) * QW_LDV + r0 + q4];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
          const double a0 = Vs[(16 * mi + g) * QW_LDV + r0 + q4];
          const double a1 = Vs[(16 * mi + g + 8) * QW_LDV + r0 + q4];
          dmma_16x8x4(acc[mi], a0, a1, b0);
        }
      }
      double* G = Gp + (warp >> 2) * 32 * QW_LDS;
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int e = 0; e < 4; ++e) G[(16 * mi + g + 8 * (e >> 1)) * QW_LDS + c0 + 2 * q4 + (e & 1)] = acc[mi][e];
    }
    __syncthreads();
    // T, blockwise: the four diagonal 8 x 8 blocks by the larft recurrence (warps 0-3 in parallel), then
    // T_AB = -T_A (V_A' V_B) T_B for the block pairs (0,1), (2,3) and then ({0,1}, {2,3})  [Q_A Q_B = I - [V_A V_B]
    // [T_A, -T_A V_A'V_B T_B; 0, T_B] [V_A V_B]'].  (V'V: the two K-half partials summed into Gp[0] first.)
    for (int idx = t; idx < 32 * 32; idx += QW_NT) {
      const int i = idx >> 5, j = idx & 31;
      Gp[i * QW_LDS + j] += Gp[32 * QW_LDS + i * QW_LDS + j];
      Ts[i * QW_LDS + j] = 0.0;
    }
    __syncthreads();
    double* W = Gp + 32 * QW_LDS;  // scratch for the off-diagonal blocks (the second partial is consumed)
    if (warp < 4) {
      const int I0 = 8 * warp;
      for (int jj = 0; jj < 8; ++jj) {
        const int j = I0 + jj;
        if (lane < 8 && j < n) {
          const int i = I0 + lane;
          double v = 0.0;
          if (i < j) {
            double s0 = 0.0;
            for (int l = i; l < j; ++l) s0 += Ts[i * QW_LDS + l] * Gp[l * QW_LDS + j];
            v = -bh[j] * s0;
          } else if (i == j) {
            v = bh[j];
          }
          Ts[i * QW_LDS + j] = v;
        }
        __syncwarp();
      }
    }
    __syncthreads();
    // level 1 (warps 0, 1): blocks (A, B) = (0, 1), (2, 3): W = G_AB T_B, then T_AB = -T_A W
    if (warp < 2) {
      const int A0 = 16 * warp, B0 = A0 + 8;
      for (int e = lane; e < 64; e += 32) {
        const int i = e >> 3, j = e & 7;
        double s0 = 0.0;
        for (int l = 0; l <= j; ++l) s0 += Gp[(A0 + i) * QW_LDS + B0 + l] * Ts[(B0 + l) * QW_LDS + B0 + j];
        W[(A0 + i) * QW_LDS + B0 + j] = s0;
      }
      __syncwarp();
      for (int e = lane; e < 64; e += 32) {
        const int i = e >> 3, j = e & 7;
        double s0 = 0.0;
        for (int l = i; l < 8; ++l) s0 += Ts[(A0 + i) * QW_LDS + A0 + l] * W[(A0 + l) * QW_LDS + B0 + j];
        Ts[(A0 + i) * QW_LDS + B0 + j] = -s0;
      }
    }
    __syncthreads();
    // level 2 (all warps): A = columns 0..15, B = 16..31: W = G_AB T_B (16 x 16), T_AB = -T_A W
    {
      const int i = t >> 4, j = t & 15;  // 256 threads = 16 x 16 outputs
      double s0 = 0.0;
      for (int l = 0; l <= j; ++l) s0 += Gp[i * QW_LDS + 16 + l] * Ts[(16 + l) * QW_LDS + 16 + j];
      W[i * QW_LDS + 16 + j] = s0;
      __syncthreads();
      double s1 = 0.0;
      for (int l = i; l < 16; ++l) s1 += Ts[i * QW_LDS + l] * W[l * QW_LDS + 16 + j];
      Ts[i * QW_LDS + 16 + j] = -s1;
    }
    __syncthreads();
    // Y = V_top' C and then Z = -(T Y), both 32 x 32 x 32 on the DMMA: warp w -> tile (w >> 2, w & 3)
    {
      const int mi = warp >> 2, ni = warp & 3;
      double y[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const double a0 = Vs[(16 * mi + g) * QW_LDV + 4 * kk + q4];      // V'[i][r] = V[r][i], rows r < 32
        const double a1 = Vs[(16 * mi + g + 8) * QW_LDV + 4 * kk + q4];
        const double b0 = Cs[(4 * kk + q4) * QW_LDS + 8 * ni + g];
        dmma_16x8x4(y, a0, a1, b0);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) Ys[(16 * mi + g + 8 * (e >> 1)) * QW_LDS + 8 * ni + 2 * q4 + (e & 1)] = y[e];
      __syncthreads();
      double z[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const double a0 = Ts[(16 * mi + g) * QW_LDS + 4 * kk + q4];
        const double a1 = Ts[(16 * mi + g + 8) * QW_LDS + 4 * kk + q4];
        const double b0 = Ys[(4 * kk + q4) * QW_LDS + 8 * ni + g];
        dmma_16x8x4(z, a0, a1, b0);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) Zs[(16 * mi + g + 8 * (e >> 1)) * QW_LDS + 8 * ni + 2 * q4 + (e & 1)] = -z[e];
    }
    __syncthreads();
    // E = [C; 0] + V Z: warp w -> rows [32 w, +32), all 32 columns
    double acc[2][4][4];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int r = 32 * warp + 16 * mi + g + 8 * (e >> 1);
          const int c = 8 * ni + 2 * q4 + (e & 1);
          acc[mi][ni][e] = (r < 32) ? Cs[r * QW_LDS + c] : 0.0;
        }
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      double a0[2], a1[2], b0[4];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        a0[mi] = Vs[(4 * kk + q4) * QW_LDV + 32 * warp + 16 * mi + g];
        a1[mi] = Vs[(4 * kk + q4) * QW_LDV + 32 * warp + 16 * mi + g + 8];
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) b0[ni] = Zs[(4 * kk + q4) * QW_LDS + 8 * ni + g];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma_16x8x4(acc[mi][ni], a0[mi], a1[mi], b0[ni]);
    }
    __syncthreads();  // every warp is done reading V: E goes through the same buffer
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int r = 32 * warp + 16 * mi + g + 8 * (e >> 1);
          const int c = 8 * ni + 2 * q4 + (e & 1);
          Vs[c * QW_LDV + r] = acc[mi][ni][e];
        }
    __syncthreads();
    if (t < L)
      for (int j = 0; j < n; ++j) I.refl[(int64_t)j * I.ldr + I.rr0 + t] = Vs[j * QW_LDV + t];
  }
}

// ------------------------------------------------------------------------------------------
// Counter-based normal generator for synthetic inputs: Philox4x32-10 on (element, stream) keyed
// by the seed, Box-Muller on two 53-bit uniforms (u1 in (0,1]).  Element e of a rows x cols
// matrix is e = col * rows + row, independent of the leading dimension.
__device__ __forceinline__ void philox(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t h0 = (uint32_t)(p0 >> 32), l0 = (uint32_t)p0;
    const uint32_t h1 = (uint32_t)(p1 >> 32), l1 = (uint32_t)p1;
    const uint32_t n0 = h1 ^ c[1] ^ k0, n2 = h0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = l1; c[2] = n2; c[3] = l0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// Rows [row0, row0 + rows) of the rows_total x cols matrix: any row sharding draws the same values.
__global__ void k_synth_normal(double* out, int64_t rows, int64_t cols, int64_t ld, int64_t row0, int64_t rows_total,
                               uint64_t seed, uint64_t stream) {
  const int64_t total = rows * cols;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = idx / rows, row = idx - col * rows;
    const int64_t e = col * rows_total + row0 + row;  // logical element of the global matrix
    const int64_t pidx = e >> 1;
    uint32_t c[4] = {(uint32_t)pidx, (uint32_t)(pidx >> 32), (uint32_t)stream, (uint32_t)(stream >> 32)};
    philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const uint64_t a = ((uint64_t)c[0] << 32) | c[1];
    const uint64_t bb = ((uint64_t)c[2] << 32) | c[3];
    const double u1 = ((double)(a >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = (double)(bb >> 11) * 0x1.0p-53;
    const double rad = sqrt(-2.0 * log(u1));
    double sv, cv;
    sincospi(2.0 * u2, &sv, &cv);
    out[col * ld + row] = (e & 1) ? rad * sv : rad * cv;
  }
}

// y_b += X_b beta_b (row sums, ascending j) for the synthetic response.
__global__ void k_add_xbeta(int G, int64_t M, const int* nb, const int64_t* p0, const double* X, int64_t ldx,
                            const double* beta, double* Y, int64_t ldy) {
  const int b = blockIdx.y;
  const int n = nb[b];
  const int64_t pb = p0[b];
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < M; k += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < n; ++j) s = s + X[(pb + j) * ldx + k] * beta[pb + j];
    Y[(int64_t)b * ldy + k] = s + Y[(int64_t)b * ldy + k];
  }
}

// Rank check on the final R diagonal (linalg.cpp:55-63): flag[b] = 1 when deficient.
__global__ void k_rank_check(Geo g, const double* R, int* flags) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.G) return;
  const int n = g.nb[b];
  const double* Rb = R + g.r0[b];
  double mx = 0.0, mn = __longlong_as_double(0x7ff0000000000000LL);
  for (int k = 0; k < n; ++k) {
    const double d = fabs(Rb[k + (int64_t)k * n]);
    mx = dmax_std(mx, d);
    mn = (d < mn) ? d : mn;
  }
  flags[b] = (mx == 0.0 || mn <= 1e-10 * mx) ? 1 : 0;
}

// out[i] = a[i] - b[i] style helpers ---------------------------------------------------------
// r = (sw + X z) - y   (pcg.cpp:69-70); X z row sums per block in ascending j.
__global__ void k_init_residual(Geo g, const double* X, int64_t ldx, const double* z, const double* sw,
                                const double* Y, int64_t ldy, double* r) {
  const int b = blockIdx.y;
  const int nb = g.nb[b];
  const int64_t p0 = g.p0[b];
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < g.ldm; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t off = (int64_t)b * g.ldm + k;
    double xz = 0.0;
    double yv = 0.0;
    if (k < g.M) {
      if (X)  // X == nullptr: z = 0 (X z = 0 exactly), X not read
        for (int j = 0; j < nb; ++j) xz = xz + X[(p0 + j) * ldx + k] * z[p0 + j];
      yv = Y[(int64_t)b * ldy + k];
    }
    r[off] = (sw[off] + xz) - yv;
  }
}

__global__ void k_axpy_sub(double* w, const double* corr, int64_t count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    w[i] -= corr[i];
}

__global__ void k_fill(double* p, double v, int64_t count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// Frobenius norm partials of X (storage order of the dense embed: columns, rows; pcg.cpp:60).
__global__ void k_sumsq_cols(const double* X, int64_t ldx, int64_t M, int64_t ncols, double* partials) {
  double s = 0.0;
  for (int64_t j = blockIdx.x; j < ncols; j += gridDim.x)
    for (int64_t k = threadIdx.x; k < M; k += blockDim.x) {
      const double v = X[j * ldx + k];
      s += v * v;
    }
  __shared__ double red[NT / 32];
  double v1[1] = {s};
  block_sum<1>(v1, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = v1[0];
}

__global__ void k_sum1(const double* partials, int count, double* out) {
  double v[1] = {0.0};
  for (int i = threadIdx.x; i < count; i += blockDim.x) v[0] += partials[i];
  __shared__ double red[32];
  block_sum<1>(v, red);
  if (threadIdx.x == 0) *out = v[0];
}

}  // namespace glsgpu
