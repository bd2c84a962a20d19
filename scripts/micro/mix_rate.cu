// Microbenchmark (development aid): what FP64 work in side warps costs a DMMA stream on the same SM.
// 8 math warps issue mma.sync.m16n8k4.f64 (16 independent accumulator blocks each, as pass A's k_kron_mma);
// E side warps do, per "chunk" (32 DMMAs per math warp, one CTA barrier), either nothing, N DFMAs per thread
// (independent or chained), or the same element work as DMMAs.  Prints the math warps' DMMA rate.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mix_rate mix_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a0), "d"(a1), "d"(b0));
}
template <int MODE, int N>
__global__ void k(double* out, int chunks, int sync) {
  const int warp = threadIdx.x >> 5;
  double s = 0.0;
  if (warp < 8) {
    double c[16][4], a[8], b[4];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
    for (int i = 0; i < 4; ++i) b[i] = 1e-3 * i + 0.5;
    for (int t = 0; t < 16; ++t)
      for (int i = 0; i < 4; ++i) c[t][i] = 0.0;
    for (int ch = 0; ch < chunks; ++ch) {
      if (sync) __syncthreads();
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int t = 0; t < 16; ++t) dmma(c[t], a[t & 7], a[(t + 1) & 7], b[t & 3]);
    }
    for (int t = 0; t < 16; ++t)
      for (int i = 0; i < 4; ++i) s += c[t][i];
  } else {
    double x[16], m = 1.0000001 + threadIdx.x * 1e-9;
    for (int i = 0; i < 16; ++i) x[i] = i + threadIdx.x;
    double c[4][4] = {};
    for (int ch = 0; ch < chunks; ++ch) {
      if (sync) __syncthreads();
      if (MODE == 1) {
#pragma unroll
        for (int i = 0; i < N; ++i) x[i & 15] = __fma_rn(x[i & 15], m, 0.5);
      } else if (MODE == 2) {
#pragma unroll
        for (int i = 0; i < N; ++i) x[0] = __fma_rn(x[0], m, 0.5);
      } else if (MODE == 3) {
#pragma unroll
        for (int i = 0; i < N; ++i) dmma(c[i & 3], x[i & 15], x[(i + 1) & 15], m);
      }
    }
    for (int i = 0; i < 16; ++i) s += x[i];
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) s += c[i][j];
  }
  if (s == 12345.0) out[0] = s;
}
template <int MODE, int N>
void run(int ew, int sms, int sync, const char* what) {
  double* o;
  cudaMalloc(&o, 8);
  const int chunks = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<MODE, N><<<sms, (8 + ew) * 32>>>(o, 10, sync);
  cudaEventRecord(e0);
  k<MODE, N><<<sms, (8 + ew) * 32>>>(o, chunks, sync);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 16 * 8 * 4 * 32.0 * chunks * 8 * sms;
  printf("%-44s side warps %d sync %d: %.2f ms, math %.1f TFLOP/s (%s)\n", what, ew, sync, ms, flops / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(o);
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int sync = 1; sync >= 0; --sync) {
    run<0, 0>(3, sms, sync, "idle side warps");
    run<1, 16>(3, sms, sync, "16 independent DFMA / thread / chunk");
    run<2, 16>(3, sms, sync, "16 chained DFMA / thread / chunk");
    run<1, 8>(3, sms, sync, "8 independent DFMA");
    run<1, 4>(3, sms, sync, "4 independent DFMA");
    run<3, 11>(3, sms, sync, "11 DMMA / side warp / chunk (same work)");
    run<3, 4>(3, sms, sync, "4 DMMA / side warp / chunk");
    run<1, 16>(7, sms, sync, "16 independent DFMA, 7 side warps");
    run<1, 7>(7, sms, sync, "7 independent DFMA, 7 side warps (same work)");
  }
  return 0;
}
