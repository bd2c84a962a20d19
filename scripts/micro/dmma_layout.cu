#include <cstdio>
#include <cmath>
__global__ void k(const double* A, const double* B, double* C) {  // A 16x4 row-major, B 4x8 row-major, C 16x8 row-major
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a0 = A[g * 4 + t], a1 = A[(g + 8) * 4 + t], b0 = B[t * 8 + g];
  double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3) : "d"(a0), "d"(a1), "d"(b0));
  C[g * 8 + 2 * t] = c0; C[g * 8 + 2 * t + 1] = c1; C[(g + 8) * 8 + 2 * t] = c2; C[(g + 8) * 8 + 2 * t + 1] = c3;
}
int main() {
  double hA[64], hB[32], hC[128], ref[128];
  for (int i = 0; i < 64; ++i) hA[i] = sin(i * 1.3) + 0.1 * i;
  for (int i = 0; i < 32; ++i) hB[i] = cos(i * 0.7) - 0.05 * i;
  for (int r = 0; r < 16; ++r) for (int c = 0; c < 8; ++c) { double s = 0; for (int k = 0; k < 4; ++k) s = fma(hA[r*4+k], hB[k*8+c], s); ref[r*8+c] = s; }
  double *A, *B, *C; cudaMalloc(&A, 512); cudaMalloc(&B, 256); cudaMalloc(&C, 1024);
  cudaMemcpy(A, hA, 512, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, 256, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(A, B, C); cudaMemcpy(hC, C, 1024, cudaMemcpyDeviceToHost);
  double md = 0; int exact = 0;
  for (int i = 0; i < 128; ++i) { md = fmax(md, fabs(hC[i] - ref[i])); exact += hC[i] == ref[i]; }
  printf("m16n8k4 layout: max |diff| = %.3e, bitwise-equal to sequential fma: %d / 128\n", md, exact);
  // accumulation order probe: c = 1 + (1e16 * 1) + (-1e16 * 1) + ... 
  return 0;
}
