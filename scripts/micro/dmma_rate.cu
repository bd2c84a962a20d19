// Microbenchmark (development aid): FP64 tensor-core (legacy mma.sync DMMA) throughput on this GPU,
// against the DFMA rate of dfma_rate.cu.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dmma_rate dmma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int SHAPE>  // 0: m8n8k4, 1: m16n8k4, 2: m16n8k8, 3: m16n8k16
__global__ void k(double* out, int iters) {
  double a[8], b[4], c[8][4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1e-3 * i + 0.5;
  for (int t = 0; t < 8; ++t)
    for (int i = 0; i < 4; ++i) c[t][i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (SHAPE == 0)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a[t]), "d"(b[t & 3]));
      else if (SHAPE == 1)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                     : "d"(a[t]), "d"(a[(t + 1) & 7]), "d"(b[t & 3]));
      else if (SHAPE == 2)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                     : "d"(a[t]), "d"(a[(t + 1) & 7]), "d"(a[(t + 2) & 7]), "d"(a[(t + 3) & 7]), "d"(b[t & 3]),
                       "d"(b[(t + 1) & 3]));
      else
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
            "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
            : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
            : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
              "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
  for (int t = 0; t < 8; ++t)
    for (int i = 0; i < 4; ++i) s += c[t][i];
  if (s == 12345.0) out[0] = s;
}
template <int SHAPE>
void run(int warps, int sms) {
  double* o;
  cudaMalloc(&o, 8);
  const int iters = 4000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<SHAPE><<<sms, warps * 32>>>(o, 10);
  cudaEventRecord(e0);
  k<SHAPE><<<sms, warps * 32>>>(o, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const int mnk[4][3] = {{8, 8, 4}, {16, 8, 4}, {16, 8, 8}, {16, 8, 16}};
  const double flops = 2.0 * mnk[SHAPE][0] * mnk[SHAPE][1] * mnk[SHAPE][2] * 8.0 * iters * warps * sms;
  printf("m%dn%dk%d warps/SM=%d: %.2f ms, %.1f TFLOP/s (%s)\n", mnk[SHAPE][0], mnk[SHAPE][1], mnk[SHAPE][2], warps, ms,
         flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(o);
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8, 16}) {
    run<0>(w, sms);
    run<1>(w, sms);
    run<2>(w, sms);
    run<3>(w, sms);
  }
  return 0;
}
