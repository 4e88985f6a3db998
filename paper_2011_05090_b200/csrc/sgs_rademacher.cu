// Rademacher sketch generated on the device: column j of the
// reference's unscaled +-1 matrix is Philox(key = (seed << 64) | j)
// .integers(0, 2, size=k) (sketch.py:153-158).  numpy's Philox is Random123
// Philox4x64-10 with the counter incremented before each block of four 64-bit
// outputs; next_uint32 hands out the low then the high half of each output,
// and integers(0, 2) is Lemire's bounded draw on one uint32, i.e. its top
// bit.  So bit r of column j is bit 31 of the r-th 32-bit draw: reproduced
// here bit for bit, one thread per column, and stored packed (row j of an
// n x kw uint32 array, bit r % 32 of word r / 32 set = +1).  At 1 bit per
// entry the operator is 64x smaller than the fp64 Theta^T stream (7.5 MB at
// k = 600, n = 1e5: L2-resident) and costs no host construction.
//
// The partial sketches use the dense chunking (dense_nparts_host / chunk_begin)
// and the same per-output chains in ascending row order as the fp64 dense
// kernels, so with +-1 entries they are bit-identical to them.

#include "sgs_common.cuh"

namespace sgs {

constexpr uint64_t kPhM0 = 0xD2E7470EE14C6C93ull, kPhM1 = 0xCA5A826395121157ull;
constexpr uint64_t kPhW0 = 0x9E3779B97F4A7C15ull, kPhW1 = 0xBB67AE8584CAA73Bull;

__device__ __forceinline__ void philox4x64_10(uint64_t (&c)[4], uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += kPhW0;
      k1 += kPhW1;
    }
    const uint64_t lo0 = kPhM0 * c[0], hi0 = __umul64hi(kPhM0, c[0]);
    const uint64_t lo1 = kPhM1 * c[2], hi1 = __umul64hi(kPhM1, c[2]);
    const uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
  }
}

__global__ void __launch_bounds__(128)
rademacher_bits_kernel(uint64_t seed, int64_t col0, int64_t n, int k, int kw,
                       uint32_t* __restrict__ bits) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const uint64_t key0 = (uint64_t)(col0 + j), key1 = seed;
  uint64_t ctr = 0;
  uint32_t* row = bits + j * kw;
  for (int w = 0; w < kw; ++w) {
    uint32_t word = 0;
#pragma unroll
    for (int call = 0; call < 4; ++call) {  // 4 blocks x 4 outputs x 2 halves = 32 draws
      uint64_t c[4] = {++ctr, 0ull, 0ull, 0ull};
      philox4x64_10(c, key0, key1);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int b = call * 8 + q * 2;
        word |= (uint32_t)((c[q] >> 31) & 1ull) << b;        // low half: its bit 31
        word |= (uint32_t)((c[q] >> 63) & 1ull) << (b + 1);  // high half: its bit 31
      }
    }
    if (w == kw - 1 && (k & 31)) word &= (1u << (k & 31)) - 1u;
    row[w] = word;
  }
}

// partials[c][p][r] = sum_{j in chunk p, ascending} (+-1)_{j r} X[j][c]
// Grid (parts, row blocks of 256 sketch rows, columns): one sketch row per
// thread, one chain per row; a pass stages 256 chunk rows of x and the 8
// sign words of the CTA's row block in shared memory.  The word is read once
// per warp (broadcast) and the sign is applied by flipping x's sign bit, so a
// term is a shift, a logic op and a DADD.
constexpr int kRdThreads = 256;
constexpr int kRdSub = 256;                 // chunk rows staged per pass
constexpr int kRdWpb = kRdThreads / 32;     // sign words per row block

// CB columns per CTA (8 for batches such as P = Theta W): the staged sign
// word and its bit are shared by the CB chains of a sketch row.
template <typename TX, int CB>
__global__ void __launch_bounds__(kRdThreads)
rademacher_partials_kernel(const uint32_t* __restrict__ bits, int kw, int k,
                           const TX* __restrict__ X, int64_t ldx, int64_t n, int ncols,
                           int nparts, double* __restrict__ partials, const sgs_status* st) {
  __shared__ uint32_t sb[kRdSub * kRdWpb];
  __shared__ double sx[CB][kRdSub];
  pdl_enter();
  if (status_stopped(st)) return;
  const int p = blockIdx.x, c0 = blockIdx.z * CB;
  const int nc = min(CB, ncols - c0);
  const int w0 = blockIdx.y * kRdWpb;
  const int nwb = min(kRdWpb, kw - w0);
  const int r = blockIdx.y * kRdThreads + threadIdx.x;
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t r0 = (n * p) / nparts, r1 = (n * (p + 1)) / nparts;
  double acc[CB];
#pragma unroll
  for (int c = 0; c < CB; ++c) acc[c] = 0.0;
  for (int64_t j0 = r0; j0 < r1; j0 += kRdSub) {
    const int nj = (int)min((int64_t)kRdSub, r1 - j0);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kRdWpb; ++q) {  // word q of chunk row threadIdx.x
      if (threadIdx.x < nj && q < nwb)
        sb[threadIdx.x * kRdWpb + q] = __ldg(bits + (j0 + threadIdx.x) * kw + w0 + q);
    }
#pragma unroll
    for (int c = 0; c < CB; ++c)
      if (threadIdx.x < nj && c < nc) sx[c][threadIdx.x] = (double)X[(int64_t)(c0 + c) * ldx + j0 + threadIdx.x];
    __syncthreads();
    if (wl < nwb) {
#pragma unroll 4
      for (int jj = 0; jj < nj; ++jj) {
        const uint32_t wd = sb[jj * kRdWpb + wl];
        const unsigned long long neg = (unsigned long long)((~wd >> lane) & 1u) << 63;
#pragma unroll
        for (int c = 0; c < CB; ++c)  // (+-1) x: flip x's sign bit, one DADD per entry
          acc[c] += __longlong_as_double(__double_as_longlong(sx[c][jj]) ^ neg);
      }
    }
  }
  if (r < k) {
#pragma unroll
    for (int c = 0; c < CB; ++c)
      if (c < nc) partials[((int64_t)(c0 + c) * nparts + p) * k + r] = acc[c];
  }
}

int dense_nparts_of(int64_t n);  // sgs_sketch.cu: the dense chunking

extern "C" int sgs_rademacher_bits(uint64_t seed, int64_t col0, int64_t n, int k, uint32_t* bits,
                                   void* stream) {
  SGS_REQUIRE(bits && n >= 1 && k >= 1 && col0 >= 0, "rademacher_bits: bad args");
  const int kw = (k + 31) / 32;
  const unsigned blocks = (unsigned)((n + 127) / 128);
  rademacher_bits_kernel<<<blocks, 128, 0, as_stream(stream)>>>(seed, col0, n, k, kw, bits);
  return check_launch("rademacher_bits_kernel");
}

template <typename TX>
static int launch_rd(const uint32_t* bits, int kw, int k, const void* X, int64_t ldx, int ncols,
                     int64_t n, double* partials, const sgs_status* st, cudaStream_t s) {
  const int np = dense_nparts_of(n);
  const int ky = (k + kRdThreads - 1) / kRdThreads;
  if (ncols == 1)
    return check_ex(launch_ex(rademacher_partials_kernel<TX, 1>, dim3(np, ky, 1), dim3(kRdThreads),
                              0, s, 1, bits, kw, k, static_cast<const TX*>(X), ldx, n, ncols, np,
                              partials, st),
                    "rademacher_partials_kernel");
  constexpr int CB = 8;
  return check_ex(launch_ex(rademacher_partials_kernel<TX, CB>,
                            dim3(np, ky, (ncols + CB - 1) / CB), dim3(kRdThreads), 0, s, 1, bits,
                            kw, k, static_cast<const TX*>(X), ldx, n, ncols, np, partials, st),
                  "rademacher_partials_kernel");
}

extern "C" int sgs_rademacher_partials(const uint32_t* bits, int k, const void* X, int x_dtype,
                                       int64_t ldx, int ncols, int64_t n, double* partials,
                                       const sgs_status* st, void* stream) {
  SGS_REQUIRE(bits && X && partials, "rademacher_partials: null pointer");
  SGS_REQUIRE(k >= 1 && n >= 1 && ncols >= 1 && ncols <= 65535,
              "rademacher_partials: bad sizes");
  SGS_REQUIRE(ldx >= n, "rademacher_partials: ldx < n");
  const int kw = (k + 31) / 32;
  cudaStream_t s = as_stream(stream);
  if (x_dtype == SGS_F32) return launch_rd<float>(bits, kw, k, X, ldx, ncols, n, partials, st, s);
  if (x_dtype == SGS_F64) return launch_rd<double>(bits, kw, k, X, ldx, ncols, n, partials, st, s);
  set_error("rademacher_partials: bad dtype");
  return SGS_EINVAL;
}

}  // namespace sgs
