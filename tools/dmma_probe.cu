// Probe the arithmetic of the fp64 tensor-core MMA (mma.sync m8n8k4 f64, the
// DMMA SASS op) on sm_100a: writes trials of (A 8x4, B 4x8, C 8x8, D 8x8) as
// raw doubles to stdout; tools/dmma_probe.py checks D against candidate
// evaluation orders with exact rational arithmetic.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

__global__ void mma_kernel(const double* A, const double* B, const double* C, double* D, int trials) {
  const int l = threadIdx.x;
  for (int t = blockIdx.x; t < trials; t += gridDim.x) {
    const double* a = A + t * 32; const double* b = B + t * 32; const double* c = C + t * 64;
    double a0 = a[(l >> 2) * 4 + (l & 3)];          // A row-major 8x4: row l/4, col l%4
    double b0 = b[(l & 3) * 8 + (l >> 2)];          // B 4x8 (stored row-major k x n): k l%4, n l/4
    double c0 = c[(l >> 2) * 8 + (l & 3) * 2], c1 = c[(l >> 2) * 8 + (l & 3) * 2 + 1];
    double d0, d1;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
                 : "=d"(d0), "=d"(d1) : "d"(a0), "d"(b0), "d"(c0), "d"(c1));
    D[t * 64 + (l >> 2) * 8 + (l & 3) * 2] = d0;
    D[t * 64 + (l >> 2) * 8 + (l & 3) * 2 + 1] = d1;
  }
}

static double rnd(uint64_t* s) {  // wide-exponent random doubles with cancellation
  *s = *s * 6364136223846793005ULL + 1442695040888963407ULL;
  double u = ((*s >> 11) * 0x1.0p-53) * 2.0 - 1.0;
  *s = *s * 6364136223846793005ULL + 1442695040888963407ULL;
  int e = (int)((*s >> 33) % 60) - 30;
  return ldexp(u, e);
}

int main(int argc, char** argv) {
  const int trials = argc > 1 ? atoi(argv[1]) : 2000;
  size_t na = (size_t)trials * 32, nc = (size_t)trials * 64;
  double *A = (double*)malloc(na * 8), *B = (double*)malloc(na * 8), *C = (double*)malloc(nc * 8),
         *D = (double*)malloc(nc * 8);
  uint64_t s = 12345;
  for (size_t i = 0; i < na; ++i) { A[i] = rnd(&s); B[i] = rnd(&s); }
  for (size_t i = 0; i < nc; ++i) C[i] = (i % 3 == 0) ? 0.0 : rnd(&s);
  double *dA, *dB, *dC, *dD;
  cudaMalloc(&dA, na * 8); cudaMalloc(&dB, na * 8); cudaMalloc(&dC, nc * 8); cudaMalloc(&dD, nc * 8);
  cudaMemcpy(dA, A, na * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B, na * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dC, C, nc * 8, cudaMemcpyHostToDevice);
  mma_kernel<<<64, 32>>>(dA, dB, dC, dD, trials);
  if (cudaDeviceSynchronize() != cudaSuccess) { fprintf(stderr, "cuda error\n"); return 1; }
  cudaMemcpy(D, dD, nc * 8, cudaMemcpyDeviceToHost);
  fwrite(&trials, 4, 1, stdout);
  fwrite(A, 8, na, stdout); fwrite(B, 8, na, stdout); fwrite(C, 8, nc, stdout); fwrite(D, 8, nc, stdout);
  return 0;
}
