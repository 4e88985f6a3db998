// Shared-memory Sylvester FWHT building blocks (used by the stand-alone
// sketch kernel and by the fused column kernel's sketch epilogue).
#pragma once
#include "sgs_common.cuh"

namespace sgs {

// padded shared-memory index: one spare slot per 8 doubles keeps the
// radix-8 passes free of bank conflicts beyond the inherent 2 wavefronts.
__host__ __device__ __forceinline__ int pidx(int e) { return e + (e >> 3); }

template <int NB>
__device__ __forceinline__ void fwht_reg(double* v) {
  // in-register Sylvester FWHT of 2^NB values (same butterfly as fwht()).
#pragma unroll
  for (int h = 1; h < (1 << NB); h <<= 1) {
#pragma unroll
    for (int q = 0; q < (1 << NB); ++q) {
      if ((q & h) == 0) {
        double a = v[q], b = v[q + h];
        v[q] = a + b;
        v[q + h] = a - b;
      }
    }
  }
}

// One radix-2^NB pass over bits [b0, b0+NB) of a 2^LOGT tile in smem.
template <int LOGT, int NB>
__device__ __forceinline__ void fwht_pass(double* z, int b0) {
  constexpr int T = 1 << LOGT;
  constexpr int G = T >> NB;
  for (int grp = threadIdx.x; grp < G; grp += blockDim.x) {
    const int lo = grp & ((1 << b0) - 1);
    const int base = lo | ((grp >> b0) << (b0 + NB));
    double v[1 << NB];
#pragma unroll
    for (int q = 0; q < (1 << NB); ++q) v[q] = z[pidx(base + (q << b0))];
    fwht_reg<NB>(v);
#pragma unroll
    for (int q = 0; q < (1 << NB); ++q) z[pidx(base + (q << b0))] = v[q];
  }
}

// The passes of fwht_tile that remain once the top bits [B, LOGT) are done:
// the same 3-bit passes, from bit B down.
template <int LOGT, int B>
__device__ __forceinline__ void fwht_tile_from(double* z) {
  int b0 = B;
#pragma unroll
  for (int p = 0; p < (B + 2) / 3; ++p) {
    const int nb = (b0 >= 3) ? 3 : b0;
    b0 -= nb;
    if (nb == 3) fwht_pass<LOGT, 3>(z, b0);
    else if (nb == 2) fwht_pass<LOGT, 2>(z, b0);
    else fwht_pass<LOGT, 1>(z, b0);
    __syncthreads();
  }
}

template <int LOGT>
__device__ __forceinline__ void fwht_tile(double* z) {
  // passes of 3 bits from the top down (any bit order gives the transform)
  int b0 = LOGT;
#pragma unroll
  for (int p = 0; p < (LOGT + 2) / 3; ++p) {
    const int nb = (b0 >= 3) ? 3 : b0;
    b0 -= nb;
    if (nb == 3) fwht_pass<LOGT, 3>(z, b0);
    else if (nb == 2) fwht_pass<LOGT, 2>(z, b0);
    else fwht_pass<LOGT, 1>(z, b0);
    __syncthreads();
  }
}

}  // namespace sgs
