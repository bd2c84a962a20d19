// Microbenchmark (development aid): sustained FP64 DFMA / DMUL+DADD issue rate per SM on this GPU.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dfma_rate dfma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int CH, bool FMA>
__global__ void k(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i] = FMA ? __fma_rn(acc[i], a, b) : __dadd_rn(__dmul_rn(acc[i], a), b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i];
  if (s == 12345.0) out[0] = s;
}
template <int CH, bool FMA>
void run(int warps, int sms) {
  double* o; cudaMalloc(&o, 8);
  const int iters = 20000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<CH, FMA><<<sms, warps * 32>>>(o, 10, 0.999, 1e-3);
  cudaEventRecord(e0);
  k<CH, FMA><<<sms, warps * 32>>>(o, iters, 0.999, 1e-3);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double ops = (double)sms * warps * 32 * CH * iters * (FMA ? 1 : 2);
  printf("%s chains=%d warps/SM=%d: %.2f ms, %.1f G instr/s, %.1f lane-ops/clk/SM at %.0f MHz nominal\n",
         FMA ? "DFMA" : "DMUL+DADD", CH, warps, ms, ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1e3);
  cudaFree(o);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8, 16}) { run<16, true>(w, sms); run<32, true>(w, sms); }
  run<32, false>(8, sms);
  return 0;
}
