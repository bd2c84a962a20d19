// Setup factorisation as CholeskyQR2 on the FP64 tensor cores (round 2).
//
// The reference factors every block by Householder QR (SurPreconditioner ctor, structured.cpp:427-450 ->
// householder_factor / form_q_columns, linalg.cpp:24-95); what the solve consumes is an orthonormal basis Q_b of
// range(w_b X_b) and the triangular R_b with Q_b R_b = w_b X_b (pi_impl / xstar_t_impl / xstar_impl,
// structured.cpp:307-363, are invariant to the signs of R's rows).  For a tall block (M >> n_b) the Householder
// leaves are latency-bound chains of n_b dependent reflections per 256 rows (kernels.cuh, the TSQR kernels); the
// same factors come out of three streaming passes of small DMMA products:
//   pass 0  G1 = X'X                       (k_cqr_pass<.., 0>: per-item partial Grams, summed in a fixed order)
//           R1 = chol(G1), R1^-1           (k_cqr_chol<false>)
//   pass 1  Q1 = X R1^-1 -> Q, G2 = Q1'Q1  (k_cqr_pass<.., 1>)
//           R2 = chol(G2), R2^-1; R = w R2 R1; delta = max |G2 - I|   (k_cqr_chol<true>)
//   pass 2  Q = Q1 R2^-1 in place          (k_cqr_pass<.., 2>)
// CholeskyQR2 is as orthogonal and as backward stable as Householder QR whenever the first pass leaves
// |Q1'Q1 - I| < 1 (Yamamoto, Nakatsukasa, Yanagisawa, Fukaya 2015: cond(X) up to ~1e7); the second Gram measures
// exactly that, so a block whose delta n_b exceeds 1/8 (or whose Cholesky meets a non-positive pivot) raises a flag
// and the host re-factors the handle with the Householder TSQR -- which also owns the reference's rank check
// (linalg.cpp:55-63) for blocks near rank deficiency.  R has a positive diagonal here (Householder's is -sign(x_kk)).
//
// A pass is a persistent grid over (block, row-chunk) items; one producer warp moves each TR-row tile of the block
// (column segments by cp.async.bulk into a padded shared-memory ring, mbarrier expect_tx) and 16 compute warps issue
// mma.sync.m16n8k4.f64 on it.  Padded strides (TR + 4, NBP + 4: = 4 mod 16) make every fragment load conflict-free.
#pragma once

namespace glsgpu {

struct CqItem {
  int b;        // block
  int ntiles;   // TR-row tiles of this item
  int64_t r0;   // first row (a multiple of TR)
};

struct CqArgs {
  const CqItem* items;
  int nitems;
  const int* nb;            // [G] block widths
  // source: element (r, c) of block b at src + src_off[b] + (tiled ? (r / TR) TR n_b + r % TR : r) + c src_cs
  const double* src;
  const int64_t* src_off;
  int64_t src_cs;
  int src_tiled;
  int64_t src_valid;        // rows >= src_valid read as 0 (and are never touched)
  double* dst;              // MODE 1, 2: the product's destination, same addressing
  const int64_t* dst_off;
  int64_t dst_cs;
  int dst_tiled;
  int64_t dst_rows;         // rows >= dst_rows are not stored
  const double* rinv;       // MODE 1, 2: [G][NBP][NBP + 4] row-major upper-triangular inverses, zero padded
  double* gpart;            // MODE 0, 1: [nitems][NBP][NBP] partial Grams (lower triangle meaningful)
};

constexpr int CQ_CW = 16;                   // compute warps
constexpr int CQ_NT = (CQ_CW + 1) * 32;     // + the producer warp

template <int NBP>
struct CqCfg;
template <>
struct CqCfg<32> {
  static constexpr int TR = 256, STAGES = 3;
};
template <>
struct CqCfg<64> {
  static constexpr int TR = 128, STAGES = 2;
};
template <>
struct CqCfg<128> {
  static constexpr int TR = 32, STAGES = 2;
};

template <int NBP, int MODE>
constexpr size_t cq_smem_bytes() {
  constexpr int TR = CqCfg<NBP>::TR, STAGES = CqCfg<NBP>::STAGES;
  size_t d = (size_t)STAGES * NBP * (TR + 4);
  if (MODE >= 1) d += (size_t)NBP * (NBP + 4);
  if (MODE <= 1 && NBP < 128) d += (size_t)NBP * (NBP + 1);
  return d * sizeof(double);
}

__device__ __forceinline__ void cq_bar_compute() { asm volatile("bar.sync 1, %0;" ::"n"(CQ_CW * 32) : "memory"); }

// Product rows of one warp that owns 16 rows and every column of the tile (NBP = 32): column blocks in pairs, last
// pair first.  A pair reads only the tile columns up to its own (Rinv is upper triangular), so with WRITE_BACK its
// product goes back into the tile (the tile becomes Q1 in place, for this warp's Gram slice) before the pairs below
// it are formed -- 8 live accumulators.  FULL: n = 4 K4 = 8 ANW and every row is stored (no guards, constant bounds).
template <int LDT, int LDB, int ANW, bool WRITE_BACK, bool FULL>
__device__ __forceinline__ void cq_apply_own(double* T, const double* Rv, int am0, int g, int q4, int K4, int n,
                                             double* dp, int64_t cs, int64_t rlim) {
  double* dl = dp + (int64_t)(2 * q4) * cs + am0 + g;  // this lane's (row g, column 2 q4) of column block 0
#pragma unroll
  for (int grp = ANW / 2 - 1; grp >= 0; --grp) {
    const int nb0 = 2 * grp;
    double acc[2][4];
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[ni][e] = 0.0;
    const int k1 = FULL ? 2 * nb0 + 2 : min(K4, 2 * nb0 + 2), k2 = FULL ? 2 * nb0 + 4 : min(K4, 2 * nb0 + 4);
    // (FULL: the bounds are compile-time constants after the pair loop is unrolled, so these loops unroll too)
#pragma unroll
    for (int kk = 0; kk < k1; ++kk) {
      const double* tp = T + (4 * kk + q4) * LDT + am0 + g;
      const double a0 = tp[0], a1 = tp[8];
      const double* bp = Rv + (4 * kk + q4) * LDB + 8 * nb0 + g;
      dmma_16x8x4(acc[0], a0, a1, bp[0]);
      dmma_16x8x4(acc[1], a0, a1, bp[8]);
    }
#pragma unroll
    for (int kk = k1; kk < k2; ++kk) {
      const double* tp = T + (4 * kk + q4) * LDT + am0 + g;
      dmma_16x8x4(acc[1], tp[0], tp[8], Rv[(4 * kk + q4) * LDB + 8 * nb0 + 8 + g]);
    }
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        double* q = dl + (int64_t)(8 * (nb0 + ni) + (e & 1)) * cs + 8 * (e >> 1);
        if (FULL) {
          stg_cs(q, acc[ni][e]);
        } else {
          const int c = 8 * (nb0 + ni) + 2 * q4 + (e & 1);
          const int row = am0 + g + 8 * (e >> 1);
          if (c < n && row < rlim) stg_cs(q, acc[ni][e]);
        }
      }
    if (WRITE_BACK) {
      __syncwarp();  // every lane's operand loads of this pair are done
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int e = 0; e < 4; ++e)
          T[(8 * (nb0 + ni) + 2 * q4 + (e & 1)) * LDT + am0 + g + 8 * (e >> 1)] = acc[ni][e];
    }
  }
  if (WRITE_BACK) __syncwarp();
}

template <int NBP, int MODE>
__global__ void __launch_bounds__(CQ_NT, 1) k_cqr_pass(CqArgs a) {
  constexpr int TR = CqCfg<NBP>::TR, STAGES = CqCfg<NBP>::STAGES;
  constexpr int LDT = TR + 4, LDB = NBP + 4, LDG = NBP + 1;
  constexpr int TILE = NBP * LDT;
  // apply: warp -> m16 row block (w % MBT) and ANW n8 column blocks from ANW (w / MBT)
  constexpr int MBT = TR / 16;
  constexpr int ANW = (NBP / 8) / (CQ_CW / MBT);
  // Gram: warp -> GMW m16 blocks from gm0, GNW n8 blocks from gn0, k-slice ks of KS (rows of the tile)
  constexpr int KS = NBP == 32 ? 16 : NBP == 64 ? 4 : 1;
  constexpr int GMW = NBP == 32 ? 2 : 1;
  constexpr int GNW = NBP == 32 ? 4 : 8;
  constexpr int KSTEPS = TR / KS / 4;  // k-steps of one warp per tile
  constexpr bool OWN_ROWS = NBP == 32;  // apply rows of a warp == its Gram k-slice (16 rows), all columns
  static_assert(MBT * (NBP / 8 / ANW) == CQ_CW, "apply warp layout");
  static_assert(!OWN_ROWS || (MBT == CQ_CW && KS == CQ_CW && TR / KS == 16), "own-rows layout");
  static_assert(KSTEPS >= 1, "gram warp layout");

  extern __shared__ __align__(128) double csm[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], rv_full, rv_empty;
  double* ring = csm;
  double* Rv = ring + STAGES * TILE;                                    // MODE >= 1
  double* gbuf = Rv + (MODE >= 1 ? NBP * LDB : 0);                      // MODE <= 1, KS > 1
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int g = lane >> 2, q4 = lane & 3;

  for (int i = t; i < STAGES * TILE; i += CQ_NT) ring[i] = 0.0;  // pad columns / rows are read (times zero)
  if (MODE <= 1 && KS > 1)
    for (int i = t; i < NBP * LDG; i += CQ_NT) gbuf[i] = 0.0;    // (the never-accumulated upper block stays 0)
  if (t == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CQ_CW);
    }
    mbar_init(&rv_full, 1);
    mbar_init(&rv_empty, CQ_CW);
    mbar_fence_init();
  }
  fence_proxy_async_smem();
  __syncthreads();

  if (warp == CQ_CW) {
    // ---------------- producer ----------------
    RingPos rp;
    int done = 0;
    for (int it = blockIdx.x; it < a.nitems; it += gridDim.x, ++done) {
      const CqItem I = a.items[it];
      const int n = a.nb[I.b];
      if (MODE >= 1) {
        if (done > 0) mbar_wait(&rv_empty, (uint32_t)((done - 1) & 1));
        if (lane == 0) {
          constexpr uint32_t bytes = NBP * LDB * sizeof(double);
          mbar_expect_tx(&rv_full, bytes);
          tma_load_1d(Rv, a.rinv + (int64_t)I.b * NBP * LDB, bytes, &rv_full);
        }
      }
      const double* sb = a.src + a.src_off[I.b];
      for (int tl = 0; tl < I.ntiles; ++tl) {
        const int64_t r = I.r0 + (int64_t)tl * TR;
        const double* sp = sb + (a.src_tiled ? (r / TR) * (int64_t)TR * n : r);
        double* T = ring + rp.slot * TILE;
        mbar_wait(&empty[rp.slot], rp.phase ^ 1u);
        if (r + TR <= a.src_valid) {
          if (lane == 0) mbar_expect_tx(&full[rp.slot], (uint32_t)(n * TR * sizeof(double)));
          __syncwarp();
          for (int c = lane; c < n; c += 32)
            tma_load_1d(T + c * LDT, sp + (int64_t)c * a.src_cs, TR * sizeof(double), &full[rp.slot]);
        } else {
          // ragged last tile of a block: guarded loads, zero rows past the end
          const int64_t v = a.src_valid - r;
          for (int idx = lane; idx < n * TR; idx += 32) {
            const int c = idx / TR, i = idx - c * TR;
            T[c * LDT + i] = i < v ? sp[(int64_t)c * a.src_cs + i] : 0.0;
          }
          fence_proxy_async_smem();  // these generic-proxy writes before a later bulk copy into the same stage
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[rp.slot]);
        }
        rp.next(STAGES);
      }
    }
    return;
  }

  // ---------------- compute warps ----------------
  const int am0 = 16 * (warp % MBT), anb0 = ANW * (warp / MBT);
  int gm0, gn0, ks;
  if (NBP == 32) {
    gm0 = 0, gn0 = 0, ks = warp;
  } else if (NBP == 64) {
    gm0 = 16 * (warp & 3), gn0 = 0, ks = warp >> 2;
  } else {
    gm0 = 16 * (warp & 7), gn0 = 64 * (warp >> 3), ks = 0;
  }
  RingPos rp;
  int done = 0;
  for (int it = blockIdx.x; it < a.nitems; it += gridDim.x, ++done) {
    const CqItem I = a.items[it];
    const int n = a.nb[I.b];
    const int K4 = (n + 3) >> 2;
    double gacc[GMW][GNW][4];
    if (MODE <= 1) {
#pragma unroll
      for (int mi = 0; mi < GMW; ++mi)
#pragma unroll
        for (int ni = 0; ni < GNW; ++ni)
#pragma unroll
          for (int e = 0; e < 4; ++e) gacc[mi][ni][e] = 0.0;
    }
    if (MODE >= 1) mbar_wait(&rv_full, (uint32_t)(done & 1));
    double* db = MODE >= 1 ? a.dst + a.dst_off[I.b] : nullptr;
    for (int tl = 0; tl < I.ntiles; ++tl) {
      const int64_t r = I.r0 + (int64_t)tl * TR;
      double* T = ring + rp.slot * TILE;
      mbar_wait(&full[rp.slot], rp.phase);
      if (MODE >= 1) {
        // product tile = T (TR x n) Rinv (n x n upper triangular): only k-steps 4 kk <= 8 nbi + 7 contribute
        double* dp = db + (a.dst_tiled ? (r / TR) * (int64_t)TR * n : r);
        const int64_t rlim = a.dst_rows - r;  // rows of this tile that exist in the destination
        if (OWN_ROWS) {
          // NBP = 32: the warp owns 16 rows and all columns (cq_apply_own); full-width blocks on a tile that lies
          // inside the destination take the unguarded instance with constant loop bounds
          if (n == NBP && rlim >= TR) cq_apply_own<LDT, LDB, ANW, MODE == 1, true>(T, Rv, am0, g, q4, K4, n, dp, a.dst_cs, rlim);
          else cq_apply_own<LDT, LDB, ANW, MODE == 1, false>(T, Rv, am0, g, q4, K4, n, dp, a.dst_cs, rlim);
        } else {
          double acc[ANW][4];
#pragma unroll
          for (int ni = 0; ni < ANW; ++ni)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[ni][e] = 0.0;
          // (segment seg covers the k-steps that first reach column block anb0 + seg: blocks below it are done)
#pragma unroll
          for (int seg = 0; seg < ANW; ++seg) {
            const int kbeg = seg == 0 ? 0 : 2 * (anb0 + seg), kend = min(K4, 2 * (anb0 + seg) + 2);
            for (int kk = kbeg; kk < kend; ++kk) {
              const double* tp = T + (4 * kk + q4) * LDT + am0 + g;
              const double a0 = tp[0], a1 = tp[8];
              const double* bp = Rv + (4 * kk + q4) * LDB + 8 * anb0 + g;
#pragma unroll
              for (int ni = seg; ni < ANW; ++ni) dmma_16x8x4(acc[ni], a0, a1, bp[8 * ni]);
            }
          }
#pragma unroll
          for (int ni = 0; ni < ANW; ++ni)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int c = 8 * (anb0 + ni) + 2 * q4 + (e & 1);
              const int row = am0 + g + 8 * (e >> 1);
              if (c < n && row < rlim) stg_cs(dp + (int64_t)c * a.dst_cs + row, acc[ni][e]);
            }
          if (MODE == 1) {
            // the tile becomes Q1 in place; the warps share rows: barriers around the overwrite
            cq_bar_compute();  // every warp has read its A operands
#pragma unroll
            for (int ni = 0; ni < ANW; ++ni)
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int c = 8 * (anb0 + ni) + 2 * q4 + (e & 1);
                const int row = am0 + g + 8 * (e >> 1);
                T[c * LDT + row] = acc[ni][e];
              }
            cq_bar_compute();
          }
        }
      }
      if (MODE <= 1) {
        // Gram of the tile: rows [ks TR / KS, +TR / KS) as the k range of this warp
#pragma unroll(MODE == 0 ? 2 : 1)
        for (int k = 0; k < KSTEPS; ++k) {
          const int rr = ks * (TR / KS) + 4 * k + q4;
          double a0[GMW], a1[GMW];
#pragma unroll
          for (int mi = 0; mi < GMW; ++mi) {
            a0[mi] = T[(gm0 + 16 * mi + g) * LDT + rr];
            a1[mi] = T[(gm0 + 16 * mi + g + 8) * LDT + rr];
          }
#pragma unroll
          for (int ni = 0; ni < GNW; ++ni) {
            const double b0 = T[(gn0 + 8 * ni + g) * LDT + rr];
#pragma unroll
            for (int mi = 0; mi < GMW; ++mi) {
              if (NBP == 32 && mi == 0 && ni >= 2) continue;  // strictly-upper 16 x 16 block: never read
              dmma_16x8x4(gacc[mi][ni], a0[mi], a1[mi], b0);
            }
          }
        }
      }
      if (MODE == 1) fence_proxy_async_smem();  // generic-proxy writes of Q1 before the next bulk copy lands here
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[rp.slot]);
      rp.next(STAGES);
    }
    if (MODE >= 1) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&rv_empty);
    }
    if (MODE <= 1) {
      double* gp = a.gpart + (int64_t)it * NBP * NBP;
      if (KS == 1) {
#pragma unroll
        for (int mi = 0; mi < GMW; ++mi)
#pragma unroll
          for (int ni = 0; ni < GNW; ++ni)
#pragma unroll
            for (int e = 0; e < 4; ++e)
              gp[(gm0 + 16 * mi + g + 8 * (e >> 1)) * NBP + gn0 + 8 * ni + 2 * q4 + (e & 1)] = gacc[mi][ni][e];
      } else {
        // k-slices added in slice order (a fixed order: the factor is deterministic run to run)
        for (int s = 0; s < KS; ++s) {
          if (ks == s) {
#pragma unroll
            for (int mi = 0; mi < GMW; ++mi)
#pragma unroll
              for (int ni = 0; ni < GNW; ++ni)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  if (NBP == 32 && mi == 0 && ni >= 2) continue;  // never accumulated, never read
                  double* p = gbuf + (gm0 + 16 * mi + g + 8 * (e >> 1)) * LDG + gn0 + 8 * ni + 2 * q4 + (e & 1);
                  *p = s == 0 ? gacc[mi][ni][e] : *p + gacc[mi][ni][e];
                }
          }
          cq_bar_compute();
        }
        for (int idx = t; idx < NBP * NBP; idx += CQ_CW * 32) gp[idx] = gbuf[(idx / NBP) * LDG + idx % NBP];
        cq_bar_compute();
      }
    }
  }
}

// Row-sharded handles: this rank's Gram of block b = its item partials summed in item order -> gloc[b] (NBP x NBP);
// the ranks' Grams are then all-gathered and k_cqr_chol adds them in rank order (every rank holds the same R).
__global__ void __launch_bounds__(256) k_cqr_sum(int NBP, const double* gpart, const int64_t* first, const int* nsrc,
                                                 double* gloc) {
  const int b = blockIdx.x;
  const int64_t nn = (int64_t)NBP * NBP;
  const double* gs = gpart + first[b] * nn;
  const int ns = nsrc[b];
  for (int idx = threadIdx.x; idx < nn; idx += 256) {
    double s = 0.0;
    for (int q = 0; q < ns; ++q) s += gs[(int64_t)q * nn + idx];
    gloc[(int64_t)b * nn + idx] = s;
  }
}

// Per block: G = sum of the partial Grams (sources src0[b], src0[b] + sstride, ... : nsrc[b] of them, in that order),
// R = chol(G) (upper, R'R = G), R^-1 into rinv[b] (row-major, ld NBP + 4, zero padded).
// FINAL = false: R -> r1[r0[b]] (n x n column-major).  FINAL = true: delta = max |G - I| (the first pass's loss of
// orthogonality) and R_out = w_b (R R1) -> rout[r0[b]] (the block's triangular factor, structured.cpp:439-447).
// flags[b] |= 1 on a non-positive pivot, 2 when delta n > 1/8 (CholeskyQR2's second pass cannot repair that).
template <bool FINAL>
__global__ void __launch_bounds__(256) k_cqr_chol(int NBP, int b0, const int* nb, const int64_t* r0off,
                                                  const double* wts, const double* gin, const int64_t* src0,
                                                  const int* nsrc, int64_t sstride, double* r1, double* rout,
                                                  double* rinv, int* flags) {
  extern __shared__ double A[];  // n x (n + 1)
  __shared__ double red[256];
  __shared__ int bad;
  const int b = b0 + blockIdx.x, t = threadIdx.x, n = nb[b], ld = n + 1;
  const int64_t nn = (int64_t)NBP * NBP;
  const double* gs = gin + src0[b] * nn;
  const int ns = nsrc[b];
  if (t == 0) bad = 0;
  for (int idx = t; idx < n * n; idx += 256) {
    const int i = idx / n, j = idx - i * n;
    if (j > i) continue;
    double s = 0.0;
    for (int q = 0; q < ns; ++q) s += gs[(int64_t)q * sstride * nn + i * NBP + j];
    A[i * ld + j] = s;
    A[j * ld + i] = s;
  }
  __syncthreads();
  int fl = 0;
  if (FINAL) {
    double d = 0.0;
    for (int idx = t; idx < n * n; idx += 256) {
      const int i = idx / n, j = idx - i * n;
      const double v = fabs(A[i * ld + j] - (i == j ? 1.0 : 0.0));
      d = (v > d || v != v) ? v : d;  // NaN propagates
    }
    red[t] = d;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
      if (t < s) {
        const double o = red[t + s];
        red[t] = (o > red[t] || o != o) ? o : red[t];
      }
      __syncthreads();
    }
    if (!(red[0] * n <= 0.125)) fl |= 2;
  }
  // Cholesky, right-looking on the upper triangle
  for (int k = 0; k < n; ++k) {
    __syncthreads();
    const double d = A[k * ld + k];
    if (!(d > 0.0) || !(d < 1.79e308)) {  // uniform across the CTA
      fl |= 1;
      break;
    }
    const double s = sqrt(d);
    __syncthreads();
    for (int j = k + t; j < n; j += 256) A[k * ld + j] = j == k ? s : A[k * ld + j] / s;
    __syncthreads();
    const int m = n - k - 1;
    for (int idx = t; idx < m * m; idx += 256) {
      const int i = k + 1 + idx / m, j = k + 1 + idx % m;
      if (j >= i) A[i * ld + j] -= A[k * ld + i] * A[k * ld + j];
    }
  }
  __syncthreads();
  double* ri = rinv + (int64_t)b * NBP * (NBP + 4);
  if (fl & 1) {
    // no factor: leave a zero inverse so the following passes stay finite; the host re-factors by TSQR
    for (int idx = t; idx < NBP * (NBP + 4); idx += 256) ri[idx] = 0.0;
    if (t == 0) flags[b] |= fl;
    return;
  }
  if (!FINAL) {
    double* R1 = r1 + r0off[b];
    for (int idx = t; idx < n * n; idx += 256) {
      const int j = idx / n, i = idx - j * n;
      R1[idx] = i <= j ? A[i * ld + j] : 0.0;
    }
  } else {
    const double* R1 = r1 + r0off[b];
    double* Ro = rout + r0off[b];
    const double w = wts[b];
    for (int idx = t; idx < n * n; idx += 256) {
      const int j = idx / n, i = idx - j * n;
      double s = 0.0;
      if (i <= j) {
        for (int l = i; l <= j; ++l) s += A[i * ld + l] * R1[l + (int64_t)j * n];
        s *= w;
      }
      Ro[idx] = s;
    }
  }
  // in-place inverse of the upper triangle, column by column (the unblocked triangular inverse)
  for (int j = 0; j < n; ++j) {
    __syncthreads();
    const double ajj = 1.0 / A[j * ld + j];
    double x = 0.0;
    if (t < j)
      for (int l = t; l < j; ++l) x += A[t * ld + l] * A[l * ld + j];
    __syncthreads();
    if (t < j) A[t * ld + j] = -ajj * x;
    else if (t == j) A[j * ld + j] = ajj;
  }
  __syncthreads();
  for (int idx = t; idx < NBP * (NBP + 4); idx += 256) {
    const int k = idx / (NBP + 4), j = idx - k * (NBP + 4);
    ri[idx] = (k <= j && j < n) ? A[k * ld + j] : 0.0;
  }
  if (t == 0 && fl) flags[b] |= fl;
}

}  // namespace glsgpu
