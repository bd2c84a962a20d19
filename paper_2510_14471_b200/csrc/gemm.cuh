// gemm.cuh -- FP64 GEMM on the FP64 tensor cores (DMMA m16n8k4) for the sur_reduce pre-pass (structured.cpp:132-178):
// the Gram W'W, the basis W V_q Lambda_q^-1/2, and the rotations basis' X_i, basis' Y.
//
// C (m x n, column-major, ld ldc) = op(A) op(B) with op(A)(i, k) = transA ? A[k + i lda] : A[i + k lda] and likewise
// for B.  64 x 64 CTA tiles, 4 warps of 32 x 32 (2 m16 x 4 n8 DMMA blocks each), 16-deep k slabs staged in shared
// memory k-major (the fragment loads are a[k][row], b[k][col]).  Split-K over gridDim.z writes per-split partial
// tiles that k_gemm_reduce sums in split order: deterministic, no floating-point atomics.  A one-off pre-pass: the
// loads are plain coalesced global loads, not a TMA pipeline.
#pragma once

namespace glsgpu {

constexpr int GM_BM = 64, GM_BN = 64, GM_BK = 16, GM_NT = 128;
constexpr int GM_LDA = GM_BM + 4, GM_LDB = GM_BN + 4;

// lower = true: only tiles that touch the lower triangle (i >= j) of a square C are computed (SYRK use)
__global__ void __launch_bounds__(GM_NT) k_gemm_dmma(int64_t m, int64_t n, int64_t k, const double* __restrict__ A,
                                                     int64_t lda, int transA, const double* __restrict__ B, int64_t ldb,
                                                     int transB, double* __restrict__ C, int64_t ldc, int64_t split_stride,
                                                     int lower) {
  __shared__ double As[GM_BK][GM_LDA];
  __shared__ double Bs[GM_BK][GM_LDB];
  const int64_t i0 = (int64_t)blockIdx.x * GM_BM, j0 = (int64_t)blockIdx.y * GM_BN;
  if (lower && j0 > i0 + GM_BM - 1) return;
  const int splits = gridDim.z, sp = blockIdx.z;
  const int64_t kchunk = ((k + splits - 1) / splits + GM_BK - 1) / GM_BK * GM_BK;
  const int64_t kb0 = (int64_t)sp * kchunk, kb1 = (kb0 + kchunk < k) ? kb0 + kchunk : k;
  double* Cp = C + (int64_t)sp * split_stride;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  double acc[2][4][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[a][b][q] = 0.0;
  for (int64_t kb = kb0; kb < kb1; kb += GM_BK) {
    // stage op(A)[i0:i0+64, kb:kb+16] and op(B)[kb:kb+16, j0:j0+64], k-major; the fast index follows memory
    for (int e = tid; e < GM_BM * GM_BK; e += GM_NT) {
      int ii, kk;
      if (!transA) { ii = e % GM_BM; kk = e / GM_BM; } else { kk = e % GM_BK; ii = e / GM_BK; }
      const int64_t gi = i0 + ii, gk = kb + kk;
      double v = 0.0;
      if (gi < m && gk < kb1) v = transA ? A[gk + gi * lda] : A[gi + gk * lda];
      As[kk][ii] = v;
    }
    for (int e = tid; e < GM_BN * GM_BK; e += GM_NT) {
      int jj, kk;
      if (transB) { jj = e % GM_BN; kk = e / GM_BN; } else { kk = e % GM_BK; jj = e / GM_BK; }
      const int64_t gj = j0 + jj, gk = kb + kk;
      double v = 0.0;
      if (gj < n && gk < kb1) v = transB ? B[gj + gk * ldb] : B[gk + gj * ldb];
      Bs[kk][jj] = v;
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < GM_BK; ks += 4) {
      double a0[2], a1[2], b0[4];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        a0[mi] = As[ks + t][wm + 16 * mi + g];
        a1[mi] = As[ks + t][wm + 16 * mi + g + 8];
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) b0[ni] = Bs[ks + t][wn + 8 * ni + g];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma_16x8x4(acc[mi][ni], a0[mi], a1[mi], b0[ni]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t gi = i0 + wm + 16 * mi + g + 8 * (q >> 1);
        const int64_t gj = j0 + wn + 8 * ni + 2 * t + (q & 1);
        if (gi < m && gj < n) Cp[gi + gj * ldc] = acc[mi][ni][q];
      }
}

// C = sum over splits of the partial tiles (split order), m x n with ld ldc (partials at ld ldc, stride)
__global__ void k_gemm_reduce(int64_t m, int64_t n, const double* __restrict__ parts, int64_t split_stride, int splits,
                              double* __restrict__ C, int64_t ldc) {
  const int64_t total = m * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / m, i = e - j * m;
    double s = 0.0;
    for (int p = 0; p < splits; ++p) s += parts[(int64_t)p * split_stride + i + j * ldc];
    C[i + j * ldc] = s;
  }
}

}  // namespace glsgpu
