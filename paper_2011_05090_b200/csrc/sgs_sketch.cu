// Sketch operators Theta x on sm_100a.
//
// P-SRHT / block-SRHT (reference: SketchOperator.apply, sketch.py:168-184,
// fwht sketch.py:90-109).  The reference pads d∘x to s = 2^L, runs a full
// Sylvester FWHT and keeps k sampled rows.  Here the Hadamard matrix is
// factorised by bits, H_s = H_{s/T} (x) H_T with T = 2^LOGT the tile size
// (high bits outer), so sampled row r = (r_h, r_l) of H_s (d∘x) equals
//     sum_h (-1)^{popcount(r_h & h)} * FWHT_T(tile_h)[r_l].
// Each CTA transforms its tiles in shared memory (radix-8 register passes),
// gathers only the k sampled low-bit rows, applies the high-bit sign and
// accumulates into a per-CTA k-vector in shared memory.  One partial per CTA
// is written; a fixed-order reduction produces y.  Padding tiles are never
// read.  Deterministic for a fixed (n_local, log2_block).

#include <cooperative_groups.h>
#include "sgs_common.cuh"
#include "sgs_fwht.cuh"

#include <cstdlib>

namespace cg = cooperative_groups;

namespace sgs {

template <typename TX>
__device__ __forceinline__ double load_as_double(const TX* p) { return (double)__ldg(p); }

constexpr int kSrhtThreads = 512;
constexpr int kSrhtMaxLogT = 12;   // 4096-row tiles (32 KB of fp64)
constexpr int kSrhtTargetCTAs = 1024;  // one tile per CTA up to 1024 tiles (4M rows)
constexpr int kSrhtCluster = 8;    // CTAs whose k-vector partials are combined through DSMEM

// SGS_SRHT_LEGACY=1: the three-pass shared-memory transform for 4096-row tiles
// too (A/B switch; the default is the two-phase register kernel below)
static bool srht_legacy() {
  static const bool v = [] {
    const char* e = getenv("SGS_SRHT_LEGACY");
    return e && atoi(e) != 0;
  }();
  return v;
}

// One CTA transforms `tiles_per_cta` consecutive tiles and accumulates the
// signed sampled entries into a shared k-vector; the 8 CTAs of a cluster then
// sum their k-vectors through distributed shared memory in rank order, each
// CTA writing 1/8 of the group partial.  Output: one k-vector per cluster.
// 4 CTAs per SM (32 registers, the tile's sign words staged in shared memory
// instead of registers): c3's 512-tile sketch of w runs in one wave of 592
// slots instead of 444 + 68, and the batched P = Theta W gains residency.
template <typename TX, int LOGT>
__global__ void __launch_bounds__(kSrhtThreads, 4)
srht_partials_kernel(const TX* __restrict__ X, int64_t ldx, int64_t n_local,
                     int64_t row0, int log2_block, const uint32_t* __restrict__ sign_bits,
                     const int32_t* __restrict__ samples, int k, int tiles_per_cta,
                     int64_t ntiles, double* __restrict__ partials,
                     const sgs_status* st, unsigned long long* tl) {
  cg::cluster_group cl = cg::this_cluster();
  constexpr int T = 1 << LOGT;
  extern __shared__ double smem[];
  double* z = smem;                       // pidx(T) entries
  double* part = smem + pidx(T) + 8;      // k entries
  int32_t* smp = reinterpret_cast<int32_t*>(part + k);  // k entries
  uint32_t* sgn = reinterpret_cast<uint32_t*>(smp + k);  // T / 32 sign words (staged path)
  const int col = blockIdx.y;
  const int ngroups = gridDim.x / kSrhtCluster;
  const TX* x = X + (int64_t)col * ldx;
  const int64_t t0 = (int64_t)blockIdx.x * tiles_per_cta;
  const int64_t t1 = min(t0 + tiles_per_cta, ntiles);
  const int64_t bmask = (int64_t(1) << log2_block) - 1;
  const bool stage_sgn = LOGT == 12 && blockDim.x == kSrhtThreads;
  // Before the dependency wait (the operator does not depend on the
  // predecessor, only x does): clear the k-vector, load the first tile's
  // sample rows and sign words.
  for (int j = threadIdx.x; j < k; j += blockDim.x) part[j] = 0.0;
  int64_t cur_blk = -1;
  if (t0 < t1) {
    cur_blk = (row0 + t0 * T) >> log2_block;
    const int32_t* sb = samples + cur_blk * (int64_t)k;
    for (int j = threadIdx.x; j < k; j += blockDim.x) smp[j] = __ldg(sb + j);
    if (stage_sgn && threadIdx.x < T / 32) {
      const int64_t lw = t0 * T + 32 * (int64_t)threadIdx.x;
      sgn[threadIdx.x] = lw < n_local ? __ldg(sign_bits + (lw >> 5)) : ~0u;
    }
  }
  pdl_enter();
  if (status_stopped(st)) return;  // uniform across the cluster: nobody writes st here
  if (tl && threadIdx.x == 0) atomicMin(tl + 12, gtimer());

  for (int64_t t = t0; t < t1; ++t) {
    const int64_t lr0 = t * T;            // first local row of the tile
    const int64_t g0 = row0 + lr0;        // first global row
    const int64_t blk = g0 >> log2_block;
    const int64_t h = (g0 & bmask) >> LOGT;
    __syncthreads();                      // previous tile's gather is done
    if (blk != cur_blk) {
      const int32_t* sb = samples + blk * (int64_t)k;
      for (int j = threadIdx.x; j < k; j += blockDim.x) smp[j] = __ldg(sb + j);
      cur_blk = blk;
    }
    bool staged = false;
    if constexpr (LOGT == 12) {
      if (blockDim.x == kSrhtThreads) {
      staged = true;
      // 8 elements per thread, strided by 512: all loads in flight at once, and
      // the 8 values differ exactly in the top 3 bits, so fwht_tile's first
      // radix-8 pass runs in registers (same butterflies, same order).
      constexpr int Q = 8;
      // the tile's 128 sign words once into shared memory (lr0 is a multiple
      // of 4096, so word w of the tile covers rows lr0 + 32 w .. + 31); the
      // first tile's were loaded before the wait
      if (t != t0 && threadIdx.x < T / 32) {
        const int64_t lw = lr0 + 32 * (int64_t)threadIdx.x;
        sgn[threadIdx.x] = lw < n_local ? __ldg(sign_bits + (lw >> 5)) : ~0u;
      }
      double v[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int64_t lr = lr0 + threadIdx.x + q * kSrhtThreads;
        v[q] = lr < n_local ? load_as_double(x + lr) : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int e = threadIdx.x + q * kSrhtThreads;
        if (((sgn[e >> 5] >> (e & 31)) & 1u) == 0u) v[q] = -v[q];
      }
      fwht_reg<3>(v);
#pragma unroll
      for (int q = 0; q < Q; ++q) z[pidx(threadIdx.x + q * kSrhtThreads)] = v[q];
      __syncthreads();
      fwht_tile_from<LOGT, LOGT - 3>(z);
      }
    }
    if (!staged) {
      for (int e = threadIdx.x; e < T; e += blockDim.x) {
        const int64_t lr = lr0 + e;
        double v = 0.0;
        if (lr < n_local) {
          v = load_as_double(x + lr);
          const uint32_t word = __ldg(sign_bits + (lr >> 5));
          if (((word >> (lr & 31)) & 1u) == 0u) v = -v;
        }
        z[pidx(e)] = v;
      }
      __syncthreads();
      fwht_tile<LOGT>(z);
    }
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
      const int32_t r = smp[j];
      const double v = z[pidx(r & (T - 1))];
      const int64_t rh = (int64_t)(r >> LOGT);
      part[j] += (__popcll(rh & h) & 1) ? -v : v;
    }
  }
  cl.sync();  // all k-vectors of the cluster are final
  const int rank = (int)cl.block_rank();
  const int j0 = (int)(((int64_t)rank * k) / kSrhtCluster);
  const int j1 = (int)(((int64_t)(rank + 1) * k) / kSrhtCluster);
  double* out = partials + ((int64_t)col * ngroups + blockIdx.x / kSrhtCluster) * k;
  for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < kSrhtCluster; ++q) s += cl.map_shared_rank(part, q)[j];
    out[j] = s;
  }
  if (tl && threadIdx.x == 0) atomicMax(tl + 13, gtimer());
  cl.sync();  // keep shared memory alive until every CTA has read it
}

// 4096-row tiles, two-phase register FWHT (the production path for LOGT = 12).
// One 64-thread CTA per tile unit.  Phase 1: thread t holds the 64 elements
// t + 64 j of the tile (j = element bits 6..11, coalesced loads, signs applied
// on load) and transforms bits 6..11 in registers; one exchange through
// shared memory (padding e + e/64: both access patterns conflict-free) gives
// it the elements 64 t + j (bits 0..5), transformed in registers as well.  So
// the 12 stages cost one shared-memory round trip instead of three radix-8
// passes, and the 64-bit adds (768 per thread per tile) are the bound.  The
// stage order (bits 6..11, then 0..5) is also the one of the fused column
// kernel's epilogue (sgs_column.cu), so with one tile per CTA both write the
// same partials bit for bit.  The transformed tile goes back to shared memory
// for the gather of the k sampled rows; the cluster of 8 CTAs sums its
// k-vectors through DSMEM in rank order, one partial per cluster, as before.
constexpr int kTileThreads = 64;
constexpr int kTileBuf = 4096 + 64;  // xidx(4096)
__device__ __forceinline__ int xidx(int e) { return e + (e >> 6); }

// A second SRHT-kind sketch with the same tile structure (the certification
// sketch Phi of the P batch, gram_schmidt.py:304-305): each tile is
// transformed a second time with Phi's signs and samples after Theta's gather,
// its values re-read from L1/L2 (not HBM) by the thread that just loaded them.
struct SrhtSecond {
  const uint32_t* sign_bits;
  const int32_t* samples;
  int k;
  int log2_block;
  double* partials;
};

template <typename TX, bool CLUSTERED, bool PAIR>
__global__ void __launch_bounds__(kTileThreads)
srht_tile_kernel(const TX* __restrict__ X, int64_t ldx, int64_t n_local, int64_t row0,
                 int log2_block, const uint32_t* __restrict__ sign_bits,
                 const int32_t* __restrict__ samples, int k, int tiles_per_cta, int64_t ntiles,
                 double* __restrict__ partials, const sgs_status* st, unsigned long long* tl,
                 SrhtSecond b2) {
  constexpr int LOGT = 12, T = 1 << LOGT;
  extern __shared__ double smem[];
  double* buf = smem;                                  // xidx(T) entries
  double* part = smem + kTileBuf;                      // k entries
  int32_t* smp = reinterpret_cast<int32_t*>(part + k);  // k entries
  double* part2 = reinterpret_cast<double*>(smp + k + (k & 1));  // PAIR: b2.k
  int32_t* smp2 = reinterpret_cast<int32_t*>(part2 + (PAIR ? b2.k : 0));
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  SGS_DCHECK(dyn_smem_offset(smp2 + (PAIR ? b2.k : 0) + 256, smem) <= dyn_smem_bytes());
  const int col = blockIdx.y;
  const TX* x = X + (int64_t)col * ldx;
  const int64_t t0 = (int64_t)blockIdx.x * tiles_per_cta;
  const int64_t t1 = min(t0 + tiles_per_cta, ntiles);
  const int64_t bmask = (int64_t(1) << log2_block) - 1;
  // the operator does not depend on the predecessor: k-vector and first
  // sample set before the dependency wait
  for (int j = t; j < k; j += kTileThreads) part[j] = 0.0;
  if constexpr (PAIR)
    for (int j = t; j < b2.k; j += kTileThreads) part2[j] = 0.0;
  int64_t cur_blk = -1, cur_blk2 = -1;
  if (t0 < t1) {
    cur_blk = (row0 + t0 * T) >> log2_block;
    const int32_t* sb = samples + cur_blk * (int64_t)k;
    for (int j = t; j < k; j += kTileThreads) smp[j] = __ldg(sb + j);
    if constexpr (PAIR) {
      cur_blk2 = (row0 + t0 * T) >> b2.log2_block;
      const int32_t* sb2 = b2.samples + cur_blk2 * (int64_t)b2.k;
      for (int j = t; j < b2.k; j += kTileThreads) smp2[j] = __ldg(sb2 + j);
    }
  }
  pdl_enter();
  if (status_stopped(st)) return;  // uniform across the cluster
  if (tl && t == 0) atomicMin(tl + 12, gtimer());
  // one sketch of the tile at lr0: load (signs on load), bits 6..11 in
  // registers, one exchange, bits 0..5, gather the sampled rows into acc
  auto tile = [&](int64_t lr0, const uint32_t* __restrict__ bits, int lb, const int32_t* sm,
                  int kk, double* acc) {
    const int64_t g0 = row0 + lr0;
    const int64_t h = (g0 & ((int64_t(1) << lb) - 1)) >> LOGT;
    double v[64];
    if (lr0 + T <= n_local) {
#pragma unroll
      for (int j = 0; j < 64; ++j) v[j] = load_as_double(x + lr0 + t + 64 * j);
    } else {
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        const int64_t lr = lr0 + t + 64 * j;
        v[j] = lr < n_local ? load_as_double(x + lr) : 0.0;
      }
    }
    // sign word of element t + 64 j: (lr0 + 64 j + 32 w) / 32, warp-uniform
    const uint32_t* sw = bits + (lr0 >> 5) + w;
#pragma unroll
    for (int j = 0; j < 64; ++j) {
      const bool in = lr0 + 64 * j + 32 * w < n_local;
      const uint32_t word = in ? __ldg(sw + 2 * j) : ~0u;
      if (((word >> lane) & 1u) == 0u) v[j] = -v[j];
    }
    fwht_reg<6>(v);                       // bits 6..11
    __syncthreads();                      // the previous gather has read buf
#pragma unroll
    for (int j = 0; j < 64; ++j) buf[xidx(t + 64 * j)] = v[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 64; ++j) v[j] = buf[xidx(64 * t + j)];
    fwht_reg<6>(v);                       // bits 0..5
    // thread t re-writes exactly the slots it read: no barrier in between
#pragma unroll
    for (int j = 0; j < 64; ++j) buf[xidx(64 * t + j)] = v[j];
    __syncthreads();
    for (int j = t; j < kk; j += kTileThreads) {
      const int32_t r = sm[j];
      SGS_DCHECK(r >= 0 && (int64_t)r < (int64_t(1) << lb));
      const double z = buf[xidx(r & (T - 1))];
      const int64_t rh = (int64_t)(r >> LOGT);
      acc[j] += (__popcll(rh & h) & 1) ? -z : z;
    }
  };
  // Batches of fp32 columns (the c1 / c4 P = Theta W): the next tile's values
  // and sign words are loaded while the current tile is transformed (64
  // registers + a 2 x 128-word sign buffer in shared memory), so a CTA's 8
  // tiles stream back to back instead of alternating HBM latency and math.
  // Same operations in the same order: bit-identical partials.
  constexpr bool PF = sizeof(TX) == 4 && !PAIR && !CLUSTERED;
  if constexpr (PF) {
    uint32_t* sgn = reinterpret_cast<uint32_t*>(smp + k + (k & 1));  // 2 x 128 words
    auto load_raw = [&](int64_t lr0, TX (&r)[64]) {
      if (lr0 + T <= n_local) {
#pragma unroll
        for (int j = 0; j < 64; ++j) r[j] = __ldg(x + lr0 + t + 64 * j);
      } else {
#pragma unroll
        for (int j = 0; j < 64; ++j) {
          const int64_t lr = lr0 + t + 64 * j;
          r[j] = lr < n_local ? __ldg(x + lr) : TX(0);
        }
      }
    };
    auto load_sgn = [&](int64_t lr0, uint32_t& s0, uint32_t& s1) {
      const int64_t w0 = (lr0 >> 5) + t, w1 = w0 + 64;  // words t and t + 64 of the tile
      s0 = (lr0 + 32 * (int64_t)t < n_local) ? __ldg(sign_bits + w0) : ~0u;
      s1 = (lr0 + 32 * (int64_t)(t + 64) < n_local) ? __ldg(sign_bits + w1) : ~0u;
    };
    TX nx[64];
    uint32_t ns0 = 0u, ns1 = 0u;
    if (t0 < t1) {
      load_raw(t0 * T, nx);
      load_sgn(t0 * T, ns0, ns1);
    }
    for (int64_t ti = t0; ti < t1; ++ti) {
      const int64_t lr0 = ti * T;
      const int64_t g0 = row0 + lr0;
      const int64_t blk = g0 >> log2_block;
      const int64_t h = (g0 & bmask) >> LOGT;
      uint32_t* sg = sgn + 128 * (int)((ti - t0) & 1);
      sg[t] = ns0;
      sg[t + 64] = ns1;
      double v[64];
#pragma unroll
      for (int j = 0; j < 64; ++j) v[j] = (double)nx[j];
      if (ti + 1 < t1) {  // in flight while this tile is transformed
        load_raw(lr0 + T, nx);
        load_sgn(lr0 + T, ns0, ns1);
      }
      __syncthreads();  // sg visible; the previous tile's gather is done with buf / smp
      if (blk != cur_blk) {
        const int32_t* sb = samples + blk * (int64_t)k;
        for (int j = t; j < k; j += kTileThreads) smp[j] = __ldg(sb + j);
        cur_blk = blk;
      }
      // sign word of element t + 64 j: word 2 j + w of the tile
#pragma unroll
      for (int j = 0; j < 64; ++j)
        if (((sg[2 * j + w] >> lane) & 1u) == 0u) v[j] = -v[j];
      fwht_reg<6>(v);                       // bits 6..11
#pragma unroll
      for (int j = 0; j < 64; ++j) buf[xidx(t + 64 * j)] = v[j];
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 64; ++j) v[j] = buf[xidx(64 * t + j)];
      fwht_reg<6>(v);                       // bits 0..5
#pragma unroll
      for (int j = 0; j < 64; ++j) buf[xidx(64 * t + j)] = v[j];
      __syncthreads();
      for (int j = t; j < k; j += kTileThreads) {
        const int32_t r = smp[j];
        SGS_DCHECK(r >= 0 && (int64_t)r < (int64_t(1) << log2_block));
        const double z = buf[xidx(r & (T - 1))];
        const int64_t rh = (int64_t)(r >> LOGT);
        part[j] += (__popcll(rh & h) & 1) ? -z : z;
      }
    }
  }
  for (int64_t ti = t0; ti < (PF ? t0 : t1); ++ti) {
    const int64_t lr0 = ti * T;
    const int64_t g0 = row0 + lr0;
    const int64_t blk = g0 >> log2_block;
    if (blk != cur_blk || (PAIR && (g0 >> b2.log2_block) != cur_blk2)) {
      __syncthreads();                    // the previous tile's gathers are done
      if (blk != cur_blk) {
        const int32_t* sb = samples + blk * (int64_t)k;
        for (int j = t; j < k; j += kTileThreads) smp[j] = __ldg(sb + j);
        cur_blk = blk;
      }
      if constexpr (PAIR) {
        const int64_t blk2 = g0 >> b2.log2_block;
        if (blk2 != cur_blk2) {
          const int32_t* sb2 = b2.samples + blk2 * (int64_t)b2.k;
          for (int j = t; j < b2.k; j += kTileThreads) smp2[j] = __ldg(sb2 + j);
          cur_blk2 = blk2;
        }
      }
    }
    tile(lr0, sign_bits, log2_block, smp, k, part);
    if constexpr (PAIR) tile(lr0, b2.sign_bits, b2.log2_block, smp2, b2.k, part2);
  }
  if constexpr (!CLUSTERED) {
    // tiles_per_cta tiles accumulated in tile order from 0.0: the cluster sum below, bit
    // for bit ((0 + z0) + z1 ... = 0 + (0 + z0) + (0 + z1) ...)
    __syncthreads();
    double* out = partials + ((int64_t)col * gridDim.x + blockIdx.x) * k;
    for (int j = t; j < k; j += kTileThreads) out[j] = part[j];
    if constexpr (PAIR) {
      double* out2 = b2.partials + ((int64_t)col * gridDim.x + blockIdx.x) * b2.k;
      for (int j = t; j < b2.k; j += kTileThreads) out2[j] = part2[j];
    }
    if (tl && t == 0) atomicMax(tl + 13, gtimer());
  } else {
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();  // all k-vectors of the cluster are final
    const int G = (int)cl.num_blocks();  // tile_group(n_local)
    const int ngroups = gridDim.x / G;
    const int rank = (int)cl.block_rank();
    const int j0 = (int)(((int64_t)rank * k) / G);
    const int j1 = (int)(((int64_t)(rank + 1) * k) / G);
    double* out = partials + ((int64_t)col * ngroups + blockIdx.x / G) * k;
    for (int j = j0 + t; j < j1; j += kTileThreads) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < G; ++q) s += cl.map_shared_rank(part, q)[j];
      out[j] = s;
    }
    if constexpr (PAIR) {
      const int p0 = (int)(((int64_t)rank * b2.k) / G);
      const int p1 = (int)(((int64_t)(rank + 1) * b2.k) / G);
      double* out2 = b2.partials + ((int64_t)col * ngroups + blockIdx.x / G) * b2.k;
      for (int j = p0 + t; j < p1; j += kTileThreads) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < G; ++q) s += cl.map_shared_rank(part2, q)[j];
        out2[j] = s;
      }
    }
    if (tl && t == 0) atomicMax(tl + 13, gtimer());
    cl.sync();  // keep shared memory alive until every CTA has read it
  }
}

// Batches of columns (one CTA per tile_group consecutive tiles of a column, no
// cluster): 256 threads per 4096-row tile, 16 values per thread, three
// register phases of four butterfly levels - bits 6..9 | 10, 11, 0, 1 | 2..5,
// the level order of srht_tile_kernel and of the column kernel's epilogue, so
// the partials are the same bits - with two exchanges through a padded tile
// (element e in slot e + e / 16: the three phases' accesses are all
// conflict-free, and every per-register slot offset is a compile-time
// immediate).  Against the 64-thread kernel's 64 values per thread: 80
// registers instead of 228, so 3 CTAs of 8 warps per SM instead of 4 of 2
// warps, and other warps' FP64 adds cover the exchange and load latencies.
// The next tile's values and sign words are loaded during the current one.
constexpr int kT3Threads = 256;
constexpr int kT3Buf = 4096 + 256;  // t3idx(4096)
__device__ __forceinline__ int t3idx(int e) { return e + (e >> 4); }

template <typename TX, int KQ>
__global__ void __launch_bounds__(kT3Threads, sizeof(TX) == 4 && KQ <= 8 ? 3 : 2)
srht_tile3_kernel(const TX* __restrict__ X, int64_t ldx, int64_t n_local, int64_t row0,
                  int log2_block, const uint32_t* __restrict__ sign_bits,
                  const int32_t* __restrict__ samples, int k, int tiles_per_cta, int64_t ntiles,
                  double* __restrict__ partials, const sgs_status* st, unsigned long long* tl) {
  constexpr int LOGT = 12, T = 1 << LOGT;
  extern __shared__ double smem[];
  double* buf = smem;                                              // kT3Buf entries
  double* part = smem + kT3Buf;                                    // k entries
  int32_t* smp = reinterpret_cast<int32_t*>(part + k);             // k entries
  uint32_t* sgn = reinterpret_cast<uint32_t*>(smp + k + (k & 1));  // 2 x 128 sign words
  const int t = threadIdx.x;
  SGS_DCHECK(dyn_smem_offset(sgn + 256, smem) <= dyn_smem_bytes());
  const int col = blockIdx.y;
  const TX* x = X + (int64_t)col * ldx;
  const int64_t t0 = (int64_t)blockIdx.x * tiles_per_cta;
  const int64_t t1 = min(t0 + tiles_per_cta, ntiles);
  const int64_t bmask = (int64_t(1) << log2_block) - 1;
  // the k-vector: entries t + 256 q in registers (KQ >= k / 256), else in
  // shared memory
  double acc[KQ > 0 ? KQ : 1];
#pragma unroll
  for (int q = 0; q < (KQ > 0 ? KQ : 1); ++q) acc[q] = 0.0;
  if constexpr (KQ == 0)
    for (int j = t; j < k; j += kT3Threads) part[j] = 0.0;
  int64_t cur_blk = -1;
  if (t0 < t1) {  // the operator does not depend on the predecessor
    cur_blk = (row0 + t0 * T) >> log2_block;
    const int32_t* sb = samples + cur_blk * (int64_t)k;
    for (int j = t; j < k; j += kT3Threads) smp[j] = __ldg(sb + j);
  }
  pdl_enter();
  if (status_stopped(st)) return;
  if (tl && t == 0) atomicMin(tl + 12, gtimer());
  // phase A: register r holds element ea + 64 r (bits 0..5 = t & 63,
  // bits 6..9 = r, bits 10..11 = t >> 6): coalesced loads; slot base + 68 r
  const int ea = (t & 63) | ((t >> 6) << 10);
  double* const pa = buf + t3idx(ea);
  // phase B: register bits 0..3 = element bits 10, 11, 0, 1, thread = bits
  // 2..9: slot base + (r >> 2) + 1088 (r & 3)
  double* const pb = buf + t3idx(t << 2);
  // phase C: register bits 0..3 = element bits 2..5, thread = bits 0, 1, 6..11:
  // slot base + 4 r + (r >> 2)
  double* const pc = buf + t3idx((t & 3) | ((t >> 2) << 6));
  const uint32_t* const sgw = sgn + (ea >> 5);  // + 2 r (+ 128 on odd tiles)
  TX nx[16];
  uint32_t ns = ~0u;
  auto load_next = [&](int64_t lr0) {
    if (lr0 + T <= n_local) {
#pragma unroll
      for (int r = 0; r < 16; ++r) nx[r] = __ldg(x + lr0 + ea + 64 * r);
    } else {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int64_t lr = lr0 + ea + 64 * r;
        nx[r] = lr < n_local ? __ldg(x + lr) : TX(0);
      }
    }
    if (t < T / 32)  // word t of the tile covers rows lr0 + 32 t .. + 31
      ns = (lr0 + 32 * (int64_t)t < n_local) ? __ldg(sign_bits + (lr0 >> 5) + t) : ~0u;
  };
  if (t0 < t1) load_next(t0 * T);
  for (int64_t ti = t0; ti < t1; ++ti) {
    const int64_t lr0 = ti * T;
    const int64_t g0 = row0 + lr0;
    const int64_t blk = g0 >> log2_block;
    const int64_t h = (g0 & bmask) >> LOGT;
    const int odd = 128 * (int)((ti - t0) & 1);
    if (t < T / 32) sgn[odd + t] = ns;
    double v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = (double)nx[r];
    if (ti + 1 < t1) load_next(lr0 + T);  // in flight during this tile
    __syncthreads();  // sign words visible; the previous tile's gather is done with buf and smp
    if (blk != cur_blk) {
      const int32_t* sb = samples + blk * (int64_t)k;
      for (int j = t; j < k; j += kT3Threads) smp[j] = __ldg(sb + j);
      cur_blk = blk;
    }
    // element ea + 64 r: sign word (ea >> 5) + 2 r, bit t & 31 (warp-uniform word)
#pragma unroll
    for (int r = 0; r < 16; ++r)
      if (((sgw[odd + 2 * r] >> (t & 31)) & 1u) == 0u) v[r] = -v[r];
    fwht_reg<4>(v);  // bits 6..9
#pragma unroll
    for (int r = 0; r < 16; ++r) pa[68 * r] = v[r];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = pb[(r >> 2) + 1088 * (r & 3)];
    fwht_reg<4>(v);  // bits 10, 11, 0, 1
    // each thread re-writes exactly the slots it read: no barrier in between
#pragma unroll
    for (int r = 0; r < 16; ++r) pb[(r >> 2) + 1088 * (r & 3)] = v[r];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = pc[4 * r + (r >> 2)];
    fwht_reg<4>(v);  // bits 2..5
#pragma unroll
    for (int r = 0; r < 16; ++r) pc[4 * r + (r >> 2)] = v[r];
    __syncthreads();
    if constexpr (KQ > 0) {
#pragma unroll
      for (int q = 0; q < KQ; ++q) {
        const int j = t + kT3Threads * q;
        if (j < k) {
          const int32_t r = smp[j];
          SGS_DCHECK(r >= 0 && (int64_t)r < (int64_t(1) << log2_block));
          const double z = buf[t3idx(r & (T - 1))];
          const int64_t rh = (int64_t)(r >> LOGT);
          acc[q] += (__popcll(rh & h) & 1) ? -z : z;
        }
      }
    } else {
      for (int j = t; j < k; j += kT3Threads) {
        const int32_t r = smp[j];
        SGS_DCHECK(r >= 0 && (int64_t)r < (int64_t(1) << log2_block));
        const double z = buf[t3idx(r & (T - 1))];
        const int64_t rh = (int64_t)(r >> LOGT);
        part[j] += (__popcll(rh & h) & 1) ? -z : z;
      }
    }
  }
  double* out = partials + ((int64_t)col * gridDim.x + blockIdx.x) * k;
  if constexpr (KQ > 0) {
#pragma unroll
    for (int q = 0; q < KQ; ++q) {
      const int j = t + kT3Threads * q;
      if (j < k) out[j] = acc[q];
    }
  } else {
    __syncthreads();
    for (int j = t; j < k; j += kT3Threads) out[j] = part[j];
  }
  if (tl && t == 0) atomicMax(tl + 13, gtimer());
}

// SGS_SRHT_TILE64=1: batches through the 64-thread srht_tile_kernel (A/B
// switch; the default is srht_tile3_kernel)
static bool srht_tile64() {
  static const bool v = [] {
    const char* e = getenv("SGS_SRHT_TILE64");
    return e && atoi(e) != 0;
  }();
  return v;
}

template <typename TX>
static size_t srht_tile_smem(int k, int k2 = 0) {
  return (size_t)(kTileBuf + k) * sizeof(double) + (size_t)(k + (k & 1)) * sizeof(int32_t) +
         (k2 > 0 ? (size_t)k2 * sizeof(double) + (size_t)k2 * sizeof(int32_t) : 0) +
         256 * sizeof(uint32_t);  // the prefetch path's sign buffer
}

// Partition of a column into tiles and partials.  4096-row tiles (the tile
// kernel): one partial per tile_group(n_local) consecutive tiles, *nctas = number of partials
// (the fused column kernel's structure).  Smaller tiles (and SGS_SRHT_LEGACY):
// tiles_per_cta tiles per CTA, one partial per 8-CTA cluster.
static void srht_geometry(int64_t n_local, int log2_block, int* logt, int64_t* ntiles,
                          int* tpc, int* nctas) {
  const int lt = log2_block < kSrhtMaxLogT ? log2_block : kSrhtMaxLogT;
  const int64_t T = int64_t(1) << lt;
  const int64_t nt = (n_local + T - 1) / T;
  if (lt == 12 && !srht_legacy()) {
    *logt = lt;
    *ntiles = nt;
    *tpc = 1;
    const int G = tile_group(n_local);
    *nctas = (int)((nt + G - 1) / G);
    return;
  }
  const int64_t per = (nt + kSrhtTargetCTAs - 1) / kSrhtTargetCTAs;
  *logt = lt;
  *ntiles = nt;
  *tpc = (int)(per < 1 ? 1 : per);
  int64_t c = (nt + *tpc - 1) / *tpc;
  c = (c + kSrhtCluster - 1) / kSrhtCluster * kSrhtCluster;
  *nctas = (int)c;
}

template <typename TX, int LOGT>
static int launch_srht_t(const void* X, int64_t ldx, int ncols, int64_t n_local, int64_t row0,
                         int log2_block, const uint32_t* sign_bits, const int32_t* samples,
                         int k, double* partials, const sgs_status* st, cudaStream_t s,
                         int tpc, int64_t ntiles, int nctas, int geom) {
  if constexpr (LOGT == 12) {
    if (!srht_legacy()) {
      // one partial per G = tile_group(n_local) consecutive tiles (nctas = partials): few
      // columns -> one tile per CTA and a DSMEM cluster sum (parallelism);
      // batches -> one CTA runs its G tiles in order (no per-tile prologue
      // or cluster exchange).  Both give the same bits.
      const size_t sm = srht_tile_smem<TX>(k);
      // geom 1: one CTA per G tiles even for one column - a grid of ntiles/G
      // CTAs leaves most SMs free, so a following LS cluster launch finds a
      // GPC and runs its pre-wait part alongside (RGMRES's sketch of w)
      const bool batch = geom == 1 || (geom == 0 && (int64_t)nctas * ncols >= 4 * (int64_t)sm_count());
      const int G = tile_group(n_local);
      if (batch && !srht_tile64()) {
        const size_t sm3 = (size_t)(kT3Buf + k) * sizeof(double) +
                           (size_t)(k + (k & 1)) * sizeof(int32_t) + 256 * sizeof(uint32_t);
        // the k-vector in registers up to k = 2048 (8 per thread), then in
        // shared memory
        auto k3 = k <= 4 * kT3Threads   ? srht_tile3_kernel<TX, 4>
                  : k <= 8 * kT3Threads ? srht_tile3_kernel<TX, 8>
                                        : srht_tile3_kernel<TX, 0>;
        if (sm3 > 48 * 1024) cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm3);
        cudaFuncSetAttribute(k3, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
        return check_ex(launch_ex(k3, dim3(nctas, ncols), dim3(kT3Threads), sm3, s, 1,
                                  static_cast<const TX*>(X), ldx, n_local, row0, log2_block,
                                  sign_bits, samples, k, G, ntiles, partials, st,
                                  debug_timeline_row()),
                        "srht_tile3_kernel");
      }
      auto kern = batch ? srht_tile_kernel<TX, false, false> : srht_tile_kernel<TX, true, false>;
      if (sm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                           cudaSharedmemCarveoutMaxShared);
      const dim3 grid(batch ? nctas : nctas * G, ncols);
      return check_ex(launch_ex(kern, grid, dim3(kTileThreads), sm, s, batch ? 1 : G,
                                static_cast<const TX*>(X), ldx, n_local, row0, log2_block,
                                sign_bits, samples, k, batch ? G : 1, ntiles, partials,
                                st, debug_timeline_row(), SrhtSecond{}),
                      "srht_tile_kernel");
    }
  }
  constexpr int T = 1 << LOGT;
  const size_t smem = (size_t)(T + T / 8 + 8 + k) * sizeof(double) + (size_t)k * sizeof(int32_t) +
                      (size_t)(T / 32) * sizeof(uint32_t);
  auto kern = srht_partials_kernel<TX, LOGT>;
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
  int threads = kSrhtThreads;
  if (T / 8 < threads) threads = (T / 8 < 64) ? 64 : T / 8;
  if (threads < 256 && k > 1024) threads = 256;
  dim3 grid(nctas, ncols);
  return check_ex(launch_ex(kern, grid, dim3(threads), smem, s, kSrhtCluster,
                            static_cast<const TX*>(X), ldx, n_local, row0, log2_block, sign_bits,
                            samples, k, tpc, ntiles, partials, st, debug_timeline_row()),
                  "srht_partials_kernel");
}

template <typename TX>
static int launch_srht(int logt, const void* X, int64_t ldx, int ncols, int64_t n_local,
                       int64_t row0, int log2_block, const uint32_t* sign_bits,
                       const int32_t* samples, int k, double* partials, const sgs_status* st,
                       cudaStream_t s, int tpc, int64_t ntiles, int nctas, int geom) {
#define SGS_SRHT_CASE(L)                                                                   \
  case L:                                                                                  \
    return launch_srht_t<TX, L>(X, ldx, ncols, n_local, row0, log2_block, sign_bits,       \
                                samples, k, partials, st, s, tpc, ntiles, nctas, geom);
  switch (logt) {
    SGS_SRHT_CASE(0) SGS_SRHT_CASE(1) SGS_SRHT_CASE(2) SGS_SRHT_CASE(3) SGS_SRHT_CASE(4)
    SGS_SRHT_CASE(5) SGS_SRHT_CASE(6) SGS_SRHT_CASE(7) SGS_SRHT_CASE(8) SGS_SRHT_CASE(9)
    SGS_SRHT_CASE(10) SGS_SRHT_CASE(11) SGS_SRHT_CASE(12)
    default:
      set_error("srht: unsupported tile log %d", logt);
      return SGS_EINVAL;
  }
#undef SGS_SRHT_CASE
}

// ---------------------------------------------------------------------------
// Dense sketch: partials[c][p][j] = sum_{r in chunk p, ascending} ThetaT[r][j] * X[r][c]
// with the chunking a pure function of n.  GEMV for one column, split-K GEMM
// for several; identical per-output FMA chains make apply_block == apply.

constexpr int kDenseMaxParts = 296;

static int dense_nparts_host(int64_t n) {
  int64_t p = (n + 31) / 32;
  if (p > kDenseMaxParts) p = kDenseMaxParts;
  if (p < 1) p = 1;
  return (int)p;
}

__device__ __forceinline__ int64_t chunk_begin(int64_t n, int nparts, int p) {
  return (n * p) / nparts;
}

template <typename TX, int QP>
__global__ void __launch_bounds__(512)
dense_gemv_kernel(const double* __restrict__ thetaT, int64_t ldt, int k,
                  const TX* __restrict__ x, int64_t n, double* __restrict__ partials,
                  const sgs_status* st) {
  pdl_enter();
  if (status_stopped(st)) return;
  const int p = blockIdx.x, nparts = gridDim.x;
  const int64_t r0 = chunk_begin(n, nparts, p), r1 = chunk_begin(n, nparts, p + 1);
  const int kp = (k + 1) >> 1;  // column pairs (ldt even, zero padded)
  double2 acc[QP];
#pragma unroll
  for (int q = 0; q < QP; ++q) acc[q] = make_double2(0.0, 0.0);
  constexpr int U = (QP <= 2) ? 8 : 4;  // rows in flight per thread
  int64_t r = r0;
  for (; r + U <= r1; r += U) {
    double xv[U];
    double2 tv[U][QP];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      xv[u] = (double)__ldg(x + r + u);
#pragma unroll
      for (int q = 0; q < QP; ++q) {
        const int jj = threadIdx.x + q * blockDim.x;
        tv[u][q] = jj < kp ? __ldg(reinterpret_cast<const double2*>(thetaT + (r + u) * ldt) + jj)
                           : make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int q = 0; q < QP; ++q) {
        acc[q].x = fma(tv[u][q].x, xv[u], acc[q].x);
        acc[q].y = fma(tv[u][q].y, xv[u], acc[q].y);
      }
    }
  }
  for (; r < r1; ++r) {
    const double xv = (double)__ldg(x + r);
#pragma unroll
    for (int q = 0; q < QP; ++q) {
      const int jj = threadIdx.x + q * blockDim.x;
      if (jj < kp) {
        const double2 tv = __ldg(reinterpret_cast<const double2*>(thetaT + r * ldt) + jj);
        acc[q].x = fma(tv.x, xv, acc[q].x);
        acc[q].y = fma(tv.y, xv, acc[q].y);
      }
    }
  }
  double* out = partials + (int64_t)p * k;
#pragma unroll
  for (int q = 0; q < QP; ++q) {
    const int jj = threadIdx.x + q * blockDim.x;
    if (2 * jj < k) out[2 * jj] = acc[q].x;
    if (2 * jj + 1 < k) out[2 * jj + 1] = acc[q].y;
  }
}

// split-K GEMM tile: 128 sketch rows (j) x 64 columns (c), 128 threads each
// owning 8 (j) x 8 (c) outputs; per output the chain is the ascending-row FMA
// of dense_gemv_kernel over the same row chunk, so P = Theta W is
// bit-identical to per-column sketches.  Operands stream through a
// kGBS-stage cp.async pipeline of kGBR-row stages (16-byte copies for the
// rows of Theta^T, element copies for the column-major W, whose part
// boundaries are not aligned).  Both operands sit row-major in shared memory
// (j resp. c contiguous), so a row's 8 + 8 operands are four 16-byte loads
// each for 64 FMAs.
constexpr int kGBJ = 128, kGBC = 64, kGBR = 16, kGBS = 3, kGBT = 128;

__device__ __forceinline__ uint32_t smem_u32a(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
template <int B>
__device__ __forceinline__ void cp_async_el(void* dst, const void* src, bool pred) {
  const int sz = pred ? B : 0;  // src-size 0: zero-fill, nothing read
  if constexpr (B == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32a(dst)), "l"(src),
                 "r"(sz) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(smem_u32a(dst)), "l"(src),
                 "n"(B), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// W rows padded by 16 bytes: the element copies of a column's 16 rows land in
// different banks
template <typename TX> __host__ __device__ constexpr int gemm_bpad() { return kGBC + 16 / (int)sizeof(TX); }

template <typename TX>
__host__ __device__ constexpr size_t dense_gemm_smem() {
  return (size_t)kGBS * kGBR * kGBJ * sizeof(double) +
         (size_t)kGBS * kGBR * gemm_bpad<TX>() * sizeof(TX);
}

template <typename TX>
__device__ __forceinline__ void load4(const TX* p, double (&v)[4]) {
  if constexpr (sizeof(TX) == 8) {
    const double2 a = *reinterpret_cast<const double2*>(p);
    const double2 b = *reinterpret_cast<const double2*>(p + 2);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  } else {
    const float4 a = *reinterpret_cast<const float4*>(p);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  }
}

template <typename TX>
__global__ void __launch_bounds__(kGBT, 2)
dense_gemm_kernel(const double* __restrict__ thetaT, int64_t ldt, int k,
                  const TX* __restrict__ X, int64_t ldx, int ncols, int64_t n,
                  double* __restrict__ partials, const sgs_status* st) {
  pdl_enter();
  if (status_stopped(st)) return;
  extern __shared__ __align__(16) unsigned char gsm_raw[];
  double (*As)[kGBR][kGBJ] = reinterpret_cast<double (*)[kGBR][kGBJ]>(gsm_raw);
  constexpr int BP = gemm_bpad<TX>();
  TX (*Bs)[kGBR][BP] = reinterpret_cast<TX (*)[kGBR][BP]>(
      gsm_raw + (size_t)kGBS * kGBR * kGBJ * sizeof(double));
  const int jt = blockIdx.x * kGBJ, ct = blockIdx.y * kGBC;
  const int p = blockIdx.z, nparts = gridDim.z;
  const int64_t r0 = chunk_begin(n, nparts, p), r1 = chunk_begin(n, nparts, p + 1);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 8 threads
  // thread outputs: j = jt + tx*4 + {0..3} and jt + 64 + tx*4 + {0..3};
  //                 c = ct + ty*4 + {0..3} and ct + 32 + ty*4 + {0..3}
  double acc[8][8];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
  const int nst = (int)((r1 - r0 + kGBR - 1) / kGBR);
  auto issue = [&](int sidx) {
    if (sidx < nst) {
      const int buf = sidx % kGBS;
      const int64_t rs = r0 + (int64_t)sidx * kGBR;
      // Theta^T: kGBR rows x kGBJ doubles, 16-byte chunks (ldt even, zero padded)
#pragma unroll
      for (int u = 0; u < kGBR * kGBJ / 2 / kGBT; ++u) {
        const int e = threadIdx.x + u * kGBT;
        const int rr = e / (kGBJ / 2), jj = 2 * (e % (kGBJ / 2));
        const bool ok = rs + rr < r1 && jt + jj < ldt;
        const double* src = ok ? thetaT + (rs + rr) * ldt + jt + jj : thetaT;
        cp_async_el<16>(&As[buf][rr][jj], src, ok);
      }
      // W: kGBR rows x kGBC columns, one element per copy (column-major source)
#pragma unroll
      for (int u = 0; u < kGBR * kGBC / kGBT; ++u) {
        const int e = threadIdx.x + u * kGBT;
        const int cc = e / kGBR, rr = e % kGBR;
        const bool ok = rs + rr < r1 && ct + cc < ncols;
        const TX* src = ok ? X + (int64_t)(ct + cc) * ldx + rs + rr : X;
        cp_async_el<sizeof(TX)>(&Bs[buf][rr][cc], src, ok);
      }
    }
    cp_async_commit();  // one group per stage slot, even when empty
  };
#pragma unroll
  for (int q = 0; q < kGBS - 1; ++q) issue(q);
  for (int sidx = 0; sidx < nst; ++sidx) {
    cp_async_wait<kGBS - 2>();
    __syncthreads();          // stage sidx landed; stage sidx-1's buffer is free
    issue(sidx + kGBS - 1);
    const int buf = sidx % kGBS;
    const int nrow = (int)min((int64_t)kGBR, r1 - (r0 + (int64_t)sidx * kGBR));
    for (int rr = 0; rr < nrow; ++rr) {  // ascending rows: the GEMV's chain
      double av[8], bv[8];
      {
        double t0[4], t1[4];
        load4<double>(&As[buf][rr][tx * 4], t0);
        load4<double>(&As[buf][rr][64 + tx * 4], t1);
#pragma unroll
        for (int q = 0; q < 4; ++q) { av[q] = t0[q]; av[4 + q] = t1[q]; }
        load4<TX>(&Bs[buf][rr][ty * 4], t0);
        load4<TX>(&Bs[buf][rr][32 + ty * 4], t1);
#pragma unroll
        for (int q = 0; q < 4; ++q) { bv[q] = t0[q]; bv[4 + q] = t1[q]; }
      }
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int j = jt + (a < 4 ? tx * 4 + a : 64 + tx * 4 + a - 4);
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const int c = ct + (b < 4 ? ty * 4 + b : 32 + ty * 4 + b - 4);
      if (j < k && c < ncols) partials[((int64_t)c * nparts + p) * k + j] = acc[a][b];
    }
  }
}

// ---------------------------------------------------------------------------
template <typename TY>
__global__ void partials_reduce_kernel(const double* __restrict__ partials, int nparts, int k,
                                       int ncols, double scale, const double* __restrict__ den,
                                       TY* __restrict__ Y, int64_t ldy, const sgs_status* st) {
  pdl_enter();
  if (status_stopped(st)) return;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)k * ncols) return;
  const int c = (int)(idx / k), j = (int)(idx % k);
  const double acc = canon_sum(partials + (int64_t)c * nparts * k + j, k, nparts);
  const double y = scale * acc;
  Y[(int64_t)c * ldy + j] = from_double<TY>(den ? y / *den : y);
}

// ---------------------------------------------------------------------------
// Stand-alone FWHT (API parity with fwht(), sketch.py:90-109): tiles of up to
// 4096 in shared memory, then radix-2 global passes over the remaining bits.
template <int LOGT>
__global__ void fwht_tile_kernel(double* X, int64_t ldx) {
  constexpr int T = 1 << LOGT;
  extern __shared__ double z[];
  double* x = X + (int64_t)blockIdx.y * ldx + (int64_t)blockIdx.x * T;
  for (int e = threadIdx.x; e < T; e += blockDim.x) z[pidx(e)] = x[e];
  __syncthreads();
  fwht_tile<LOGT>(z);
  for (int e = threadIdx.x; e < T; e += blockDim.x) x[e] = z[pidx(e)];
}

__global__ void fwht_global_pass(double* X, int64_t ldx, int64_t s, int64_t h) {
  double* x = X + (int64_t)blockIdx.y * ldx;
  const int64_t half = s >> 1;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < half;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = t & (h - 1);
    const int64_t i = ((t - lo) << 1) + lo;
    const double a = x[i], b = x[i + h];
    x[i] = a + b;
    x[i + h] = a - b;
  }
}

template <int LOGT>
static int launch_fwht_tile(double* X, int64_t ldx, int64_t ntile, int ncols, cudaStream_t s) {
  constexpr int T = 1 << LOGT;
  const size_t smem = (size_t)(T + T / 8 + 8) * sizeof(double);
  auto kern = fwht_tile_kernel<LOGT>;
  int threads = T / 8 < 32 ? 32 : (T / 8 > 512 ? 512 : T / 8);
  kern<<<dim3((unsigned)ntile, ncols), threads, smem, s>>>(X, ldx);
  return check_launch("fwht_tile_kernel");
}



}  // namespace sgs

using namespace sgs;

extern "C" int sgs_srht_nparts(int64_t n_local, int log2_block) {
  int lt, tpc, nc;
  int64_t nt;
  if (n_local < 1 || log2_block < 0 || log2_block > 40) return 0;
  srht_geometry(n_local, log2_block, &lt, &nt, &tpc, &nc);
  return (lt == 12 && !srht_legacy()) ? nc : nc / kSrhtCluster;
}

extern "C" int sgs_srht_partials_geom(const void* X, int x_dtype, int64_t ldx, int ncols,
                                      int64_t n_local, int64_t row0, int log2_block,
                                      const uint32_t* sign_bits, const int32_t* samples, int k,
                                      double* partials, int geom, const sgs_status* st,
                                      void* stream);

extern "C" int sgs_srht_partials(const void* X, int x_dtype, int64_t ldx, int ncols,
                                 int64_t n_local, int64_t row0, int log2_block,
                                 const uint32_t* sign_bits, const int32_t* samples, int k,
                                 double* partials, const sgs_status* st, void* stream) {
  return sgs_srht_partials_geom(X, x_dtype, ldx, ncols, n_local, row0, log2_block, sign_bits,
                                samples, k, partials, 0, st, stream);
}

extern "C" int sgs_srht_partials_geom(const void* X, int x_dtype, int64_t ldx, int ncols,
                                      int64_t n_local, int64_t row0, int log2_block,
                                      const uint32_t* sign_bits, const int32_t* samples, int k,
                                      double* partials, int geom, const sgs_status* st,
                                      void* stream) {
  SGS_REQUIRE(geom >= 0 && geom <= 2, "srht: bad geometry %d", geom);
  SGS_REQUIRE(X && sign_bits && samples && partials, "srht: null pointer");
  SGS_REQUIRE(n_local >= 1 && ncols >= 1 && k >= 1 && k <= 8192, "srht: bad sizes n=%lld k=%d",
              (long long)n_local, k);
  SGS_REQUIRE(log2_block >= 0 && log2_block <= 40, "srht: bad log2_block %d", log2_block);
  SGS_REQUIRE(x_dtype == SGS_F32 || x_dtype == SGS_F64, "srht: bad dtype");
  int lt, tpc, np;
  int64_t nt;
  srht_geometry(n_local, log2_block, &lt, &nt, &tpc, &np);  // np = CTAs
  SGS_REQUIRE((row0 & ((int64_t(1) << lt) - 1)) == 0, "srht: row0 %lld not tile aligned",
              (long long)row0);
  cudaStream_t s = as_stream(stream);
  if (x_dtype == SGS_F32)
    return launch_srht<float>(lt, X, ldx, ncols, n_local, row0, log2_block, sign_bits, samples,
                              k, partials, st, s, tpc, nt, np, geom);
  return launch_srht<double>(lt, X, ldx, ncols, n_local, row0, log2_block, sign_bits, samples,
                             k, partials, st, s, tpc, nt, np, geom);
}

template <typename TX>
static int launch_srht_pair(const void* X, int64_t ldx, int ncols, int64_t n_local, int64_t row0,
                            int log2_block, const uint32_t* sign_bits, const int32_t* samples,
                            int k, double* partials, SrhtSecond b2, const sgs_status* st,
                            cudaStream_t s, int64_t ntiles, int nctas) {
  const size_t sm = srht_tile_smem<TX>(k, b2.k);
  const bool batch = (int64_t)nctas * ncols >= 4 * (int64_t)sm_count();
  auto kern = batch ? srht_tile_kernel<TX, false, true> : srht_tile_kernel<TX, true, true>;
  if (sm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
  const int G = tile_group(n_local);
  const dim3 grid(batch ? nctas : nctas * G, ncols);
  return check_ex(launch_ex(kern, grid, dim3(kTileThreads), sm, s, batch ? 1 : G,
                            static_cast<const TX*>(X), ldx, n_local, row0, log2_block, sign_bits,
                            samples, k, batch ? G : 1, ntiles, partials, st,
                            debug_timeline_row(), b2),
                  "srht_tile_kernel(pair)");
}

extern "C" int sgs_srht_partials_pair(const void* X, int x_dtype, int64_t ldx, int ncols,
                                      int64_t n_local, int64_t row0, int log2_block,
                                      const uint32_t* sign_bits, const int32_t* samples, int k,
                                      double* partials, int log2_block2,
                                      const uint32_t* sign_bits2, const int32_t* samples2, int k2,
                                      double* partials2, const sgs_status* st, void* stream) {
  SGS_REQUIRE(X && sign_bits && samples && partials && sign_bits2 && samples2 && partials2,
              "srht pair: null pointer");
  SGS_REQUIRE(n_local >= 1 && ncols >= 1 && k >= 1 && k <= 8192 && k2 >= 1 && k2 <= 8192,
              "srht pair: bad sizes n=%lld k=%d k2=%d", (long long)n_local, k, k2);
  SGS_REQUIRE(log2_block >= 12 && log2_block <= 40 && log2_block2 >= 12 && log2_block2 <= 40,
              "srht pair: both sketches need 4096-row tiles (log2 blocks %d, %d)", log2_block,
              log2_block2);
  SGS_REQUIRE(!srht_legacy(), "srht pair: not available with SGS_SRHT_LEGACY");
  SGS_REQUIRE(x_dtype == SGS_F32 || x_dtype == SGS_F64, "srht pair: bad dtype");
  SGS_REQUIRE((row0 & 4095) == 0, "srht pair: row0 %lld not tile aligned", (long long)row0);
  int lt, tpc, np;
  int64_t nt;
  srht_geometry(n_local, log2_block, &lt, &nt, &tpc, &np);
  cudaStream_t s = as_stream(stream);
  const SrhtSecond b2{sign_bits2, samples2, k2, log2_block2, partials2};
  if (x_dtype == SGS_F32)
    return launch_srht_pair<float>(X, ldx, ncols, n_local, row0, log2_block, sign_bits, samples,
                                   k, partials, b2, st, s, nt, np);
  return launch_srht_pair<double>(X, ldx, ncols, n_local, row0, log2_block, sign_bits, samples,
                                  k, partials, b2, st, s, nt, np);
}

extern "C" int sgs_dense_nparts(int64_t n) { return n < 1 ? 0 : dense_nparts_host(n); }
namespace sgs {
int dense_nparts_of(int64_t n) { return dense_nparts_host(n); }
}  // namespace sgs

// ---------------------------------------------------------------------------
// Gaussian P = Theta W on the fp64 tensor cores (mma.sync m8n8k4 f64: the DMMA
// SASS op).  The contraction over the n rows is split into nsub sub-chunks
// (chunk_begin over gaussian_nsub(n) <= 152 of them, a multiple of 8); each
// CTA owns one sub-chunk and a (j, c) output tile, and its per-output chain
// is a sequence of DMMAs over ascending 4-row k-steps (the chunk's last step
// zero-padded).  The 8 CTAs of a cluster are 8 consecutive sub-chunks: they
// sum their tiles through distributed shared memory in rank order, so one
// partial per 8 sub-chunks goes to HBM (c0: 19 x k per column instead of
// the DFMA GEMM's 296 x k).  apply() (one column) runs the same kernel with an 8-column tile:
// every output element is the same chain of the same operands, so
// apply_block is bit-identical to apply whatever the tile shape.
//
// Fragments (PTX m8n8k4 .f64, lane l): A[l/4][l%4] = Theta^T[r + l%4][j + l/4],
// B[l%4][l/4] = W[r + l%4][c + l/4], D[l/4][2 (l%4) + {0,1}].
// Rows per ring stage x stages, per tile shape (SR, NS below): a block barrier
// per stage, so the 300-column batch runs 32-row stages (c0 P batch 1.742 ->
// 1.650 ms against 16 x 3), the one-column apply keeps 16 x 3 (109 us; 140 us
// with 32 x 2).  The k-steps of a chain are the same 4-row steps either way.
// Sub-chunks of the contraction (c0, 300 columns, P batch ms / apply us per
// column: 296 1.838 / 112, 152 1.742 / 109, 104 1.732 / 123, 72 1.726 / 107,
// 40 1.781 / 129; profiles/r02k_dmma_subchunks.txt).
constexpr int kMmaMaxSub = 152;

static int gaussian_nsub(int64_t n) {
  int64_t p = (n + 31) / 32;
  p = (p + kSrhtCluster - 1) / kSrhtCluster * kSrhtCluster;
  static const int max_sub = [] {  // SGS_MMA_MAXSUB (a multiple of 8): experiment override
    const char* e = getenv("SGS_MMA_MAXSUB");
    const int v = e ? atoi(e) / kSrhtCluster * kSrhtCluster : kMmaMaxSub;
    return v >= kSrhtCluster ? v : kMmaMaxSub;
  }();
  if (p > max_sub) p = max_sub;
  return (int)p;
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <int WJ, int WC, int TJ, int TC>
struct MmaTile {
  static constexpr int kThreads = 32 * WJ * WC;
  static constexpr int kJ = WJ * TJ * 8;     // Theta rows (j) per CTA
  static constexpr int kC = WC * TC * 8;     // columns (c) per CTA
  static constexpr int kAS = kJ + 4;         // padded smem row strides: the 4 rows
  static constexpr int kBS = kC + 4;         // of a k-step fall in distinct banks
};

template <typename TX, int WJ, int WC, int TJ, int TC, int SR, int NS>
__global__ void __launch_bounds__(32 * WJ * WC)
dense_mma_kernel(const double* __restrict__ thetaT, int64_t ldt, int k, const TX* __restrict__ X,
                 int64_t ldx, int ncols, int64_t n, int nsub, double* __restrict__ partials,
                 const sgs_status* st, int njt) {
  using G = MmaTile<WJ, WC, TJ, TC>;
  constexpr int kMmaStageRows = SR, kMmaStages = NS;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char mma_raw[];
  SGS_DCHECK((size_t)G::kJ * G::kC * sizeof(double) <= dyn_smem_bytes());
  double* As = reinterpret_cast<double*>(mma_raw);                              // S x 16 x kAS
  TX* Bs = reinterpret_cast<TX*>(As + (size_t)kMmaStages * kMmaStageRows * G::kAS);  // S x 16 x kBS
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wj = warp % WJ, wc = warp / WJ;
  // grid (8 x tiles, nsub / 8): a cluster is the 8 sub-chunks of one (j, c)
  // tile, and the tiles of the same 8 sub-chunks are neighbours in launch
  // order, so their rows of Theta^T and W are read from HBM once and from L2
  // by the other tiles (with the sub-chunk fastest every tile re-read them:
  // 3.7 GB of DRAM reads for 0.72 GB of operands at c0)
  const int p = blockIdx.y * kSrhtCluster + (blockIdx.x % kSrhtCluster);  // sub-chunk
  const int tile = blockIdx.x / kSrhtCluster;
  const int jt = (tile % njt) * G::kJ, ct = (tile / njt) * G::kC;
  const int64_t r0 = chunk_begin(n, nsub, p), r1 = chunk_begin(n, nsub, p + 1);
  const int nst = (int)((r1 - r0 + kMmaStageRows - 1) / kMmaStageRows);
  double acc[TJ][TC][2];
#pragma unroll
  for (int a = 0; a < TJ; ++a)
#pragma unroll
    for (int b = 0; b < TC; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  // X may be the predecessor kernel's output (a basis column, A q): wait first
  pdl_enter();
  const bool stop = status_stopped(st);  // uniform: the cluster still meets at its barriers
  auto issue = [&](int sidx) {
    if (sidx < nst) {
      const int buf = sidx % kMmaStages;
      const int64_t rs = r0 + (int64_t)sidx * kMmaStageRows;
      double* Ab = As + (size_t)buf * kMmaStageRows * G::kAS;
      TX* Bb = Bs + (size_t)buf * kMmaStageRows * G::kBS;
      for (int e = tid; e < kMmaStageRows * G::kJ / 2; e += G::kThreads) {
        const int rr = e / (G::kJ / 2), jj = 2 * (e % (G::kJ / 2));
        const bool ok = rs + rr < r1 && jt + jj < ldt;
        cp_async_el<16>(Ab + rr * G::kAS + jj, ok ? thetaT + (rs + rr) * ldt + jt + jj : thetaT, ok);
      }
      for (int e = tid; e < kMmaStageRows * G::kC; e += G::kThreads) {
        const int cc = e / kMmaStageRows, rr = e % kMmaStageRows;
        const bool ok = rs + rr < r1 && ct + cc < ncols;
        cp_async_el<sizeof(TX)>(Bb + rr * G::kBS + cc,
                                ok ? X + (int64_t)(ct + cc) * ldx + rs + rr : X, ok);
      }
    }
    cp_async_commit();
  };
  if (!stop) {
#pragma unroll
    for (int q = 0; q < kMmaStages - 1; ++q) issue(q);
    for (int sidx = 0; sidx < nst; ++sidx) {
      cp_async_wait<kMmaStages - 2>();
      __syncthreads();
      issue(sidx + kMmaStages - 1);
      const int buf = sidx % kMmaStages;
      const double* Ab = As + (size_t)buf * kMmaStageRows * G::kAS;
      const TX* Bb = Bs + (size_t)buf * kMmaStageRows * G::kBS;
#pragma unroll
      for (int ks = 0; ks < kMmaStageRows / 4; ++ks) {  // ascending 4-row k-steps
        const int rr = 4 * ks + (lane & 3);
        double a[TJ], b[TC];
#pragma unroll
        for (int tj = 0; tj < TJ; ++tj) a[tj] = Ab[rr * G::kAS + (wj * TJ + tj) * 8 + (lane >> 2)];
#pragma unroll
        for (int tc = 0; tc < TC; ++tc)
          b[tc] = (double)Bb[rr * G::kBS + (wc * TC + tc) * 8 + (lane >> 2)];
#pragma unroll
        for (int tj = 0; tj < TJ; ++tj)
#pragma unroll
          for (int tc = 0; tc < TC; ++tc) dmma(acc[tj][tc], a[tj], b[tc]);
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // stage buffers free: the output tile aliases them
  double* Ot = reinterpret_cast<double*>(mma_raw);  // kC x kJ, column c contiguous in j
#pragma unroll
  for (int tj = 0; tj < TJ; ++tj)
#pragma unroll
    for (int tc = 0; tc < TC; ++tc)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int jl = (wj * TJ + tj) * 8 + (lane >> 2);
        const int cl_ = (wc * TC + tc) * 8 + 2 * (lane & 3) + h;
        Ot[cl_ * G::kJ + jl] = acc[tj][tc][h];
      }
  cl.sync();
  if (!stop) {
    const int rank = (int)cl.block_rank();
    constexpr int kOut = G::kJ * G::kC;
    const int e0 = rank * kOut / kSrhtCluster, e1 = (rank + 1) * kOut / kSrhtCluster;
    const int np2 = nsub / kSrhtCluster, p2 = p / kSrhtCluster;
    for (int e = e0 + tid; e < e1; e += G::kThreads) {
      const int cc = e / G::kJ, jj = e % G::kJ;
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < kSrhtCluster; ++q) s += cl.map_shared_rank(Ot, q)[e];
      if (ct + cc < ncols && jt + jj < k)
        partials[((int64_t)(ct + cc) * np2 + p2) * k + jt + jj] = s;
    }
  }
  cl.sync();  // the tile stays readable until every CTA of the cluster is done
}

template <typename TX, int WJ, int WC, int TJ, int TC, int SR, int NS>
static int launch_dense_mma_t(const double* thetaT, int64_t ldt, int k, const TX* X, int64_t ldx,
                              int ncols, int64_t n, double* partials, const sgs_status* st,
                              cudaStream_t s) {
  using G = MmaTile<WJ, WC, TJ, TC>;
  constexpr int kMmaStageRows = SR, kMmaStages = NS;
  const int nsub = gaussian_nsub(n);
  const size_t stage = (size_t)kMmaStageRows * G::kAS * sizeof(double) +
                       (size_t)kMmaStageRows * G::kBS * sizeof(TX);
  size_t smem = kMmaStages * stage;
  const size_t otile = (size_t)G::kJ * G::kC * sizeof(double);
  if (otile > smem) smem = otile;
  auto kern = dense_mma_kernel<TX, WJ, WC, TJ, TC, SR, NS>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int njt = (k + G::kJ - 1) / G::kJ, nct = (ncols + G::kC - 1) / G::kC;
  dim3 grid(kSrhtCluster * njt * nct, nsub / kSrhtCluster);
  return check_ex(launch_ex(kern, grid, dim3(G::kThreads), smem, s, kSrhtCluster, thetaT, ldt, k,
                            X, ldx, ncols, n, nsub, partials, st, njt),
                  "dense_mma_kernel");
}

template <typename TX>
static int launch_dense_mma(const double* thetaT, int64_t ldt, int k, const void* X, int64_t ldx,
                            int ncols, int64_t n, double* partials, const sgs_status* st,
                            cudaStream_t s) {
  const TX* x = static_cast<const TX*>(X);
  if (ncols <= 8)  // apply(): 256 (j) x 8 (c) tiles, 8 warps along j
    return launch_dense_mma_t<TX, 8, 1, 4, 1, 16, 3>(thetaT, ldt, k, x, ldx, ncols, n, partials, st, s);
  return launch_dense_mma_t<TX, 4, 2, 4, 4, 32, 2>(thetaT, ldt, k, x, ldx, ncols, n, partials, st, s);
}

// SGS_DENSE_LEGACY=1: the DFMA GEMV / split-K GEMM with 296 partials (A/B)
static bool dense_legacy() {
  static const bool v = [] {
    const char* e = getenv("SGS_DENSE_LEGACY");
    return e && atoi(e) != 0;
  }();
  return v;
}

template <typename TX>
static int launch_dense(const double* thetaT, int64_t ldt, int k, const void* X, int64_t ldx,
                        int ncols, int64_t n, double* partials, const sgs_status* st,
                        cudaStream_t s) {
  const int np = dense_nparts_host(n);
  const TX* x = static_cast<const TX*>(X);
  if (ncols == 1) {
    const int kp = (k + 1) / 2;
    int threads = ((kp + 31) / 32) * 32;
    if (threads > 512) threads = 512;
    const int qp = (kp + threads - 1) / threads;
    cudaError_t e;
    if (qp <= 1)
      e = launch_ex(dense_gemv_kernel<TX, 1>, dim3(np), dim3(threads), 0, s, 1, thetaT, ldt, k, x, n, partials, st);
    else if (qp <= 2)
      e = launch_ex(dense_gemv_kernel<TX, 2>, dim3(np), dim3(threads), 0, s, 1, thetaT, ldt, k, x, n, partials, st);
    else if (qp <= 4)
      e = launch_ex(dense_gemv_kernel<TX, 4>, dim3(np), dim3(threads), 0, s, 1, thetaT, ldt, k, x, n, partials, st);
    else if (qp <= 8)
      e = launch_ex(dense_gemv_kernel<TX, 8>, dim3(np), dim3(threads), 0, s, 1, thetaT, ldt, k, x, n, partials, st);
    else {
      set_error("dense sketch: k=%d too large", k);
      return SGS_EINVAL;
    }
    return check_ex(e, "dense_gemv_kernel");
  }
  dim3 grid((k + kGBJ - 1) / kGBJ, (ncols + kGBC - 1) / kGBC, np);
  constexpr size_t smem = dense_gemm_smem<TX>();
  cudaFuncSetAttribute(dense_gemm_kernel<TX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  return check_ex(launch_ex(dense_gemm_kernel<TX>, grid, dim3(kGBT), smem, s, 1, thetaT, ldt, k,
                            x, ldx, ncols, n, partials, st), "dense_gemm_kernel");
}

extern "C" int sgs_dense_partials(const double* thetaT, int64_t ldt, int k, const void* X,
                                  int x_dtype, int64_t ldx, int ncols, int64_t n,
                                  double* partials, const sgs_status* st, void* stream) {
  SGS_REQUIRE(thetaT && X && partials, "dense: null pointer");
  SGS_REQUIRE(k >= 1 && n >= 1 && ncols >= 1, "dense: bad sizes");
  SGS_REQUIRE(ldt >= k && (ldt % 2) == 0, "dense: ldt must be even and >= k");
  SGS_REQUIRE(((uintptr_t)thetaT & 15) == 0, "dense: thetaT must be 16-byte aligned");
  SGS_REQUIRE(x_dtype == SGS_F32 || x_dtype == SGS_F64, "dense: bad dtype");
  cudaStream_t s = as_stream(stream);
  if (!dense_legacy()) {
    if (x_dtype == SGS_F32)
      return launch_dense_mma<float>(thetaT, ldt, k, X, ldx, ncols, n, partials, st, s);
    return launch_dense_mma<double>(thetaT, ldt, k, X, ldx, ncols, n, partials, st, s);
  }
  if (x_dtype == SGS_F32) return launch_dense<float>(thetaT, ldt, k, X, ldx, ncols, n, partials, st, s);
  return launch_dense<double>(thetaT, ldt, k, X, ldx, ncols, n, partials, st, s);
}

extern "C" int sgs_gaussian_nparts(int64_t n) {
  if (n < 1) return 0;
  return dense_legacy() ? dense_nparts_host(n) : gaussian_nsub(n) / kSrhtCluster;
}

static int partials_reduce_impl(const double* partials, int nparts, int k, int ncols,
                                double scale, const double* den, void* Y, int y_dtype,
                                int64_t ldy, const sgs_status* st, void* stream);

extern "C" int sgs_partials_reduce(const double* partials, int nparts, int k, int ncols,
                                   double scale, void* Y, int y_dtype, int64_t ldy,
                                   const sgs_status* st, void* stream) {
  return partials_reduce_impl(partials, nparts, k, ncols, scale, nullptr, Y, y_dtype, ldy, st,
                              stream);
}

extern "C" int sgs_partials_reduce_div(const double* partials, int nparts, int k, int ncols,
                                       double scale, const double* den, void* Y, int y_dtype,
                                       int64_t ldy, const sgs_status* st, void* stream) {
  return partials_reduce_impl(partials, nparts, k, ncols, scale, den, Y, y_dtype, ldy, st,
                              stream);
}

static int partials_reduce_impl(const double* partials, int nparts, int k, int ncols,
                                double scale, const double* den, void* Y, int y_dtype,
                                int64_t ldy, const sgs_status* st, void* stream) {
  SGS_REQUIRE(partials && Y && nparts >= 1 && k >= 1 && ncols >= 1, "reduce: bad args");
  SGS_REQUIRE(ldy >= k, "reduce: ldy < k");
  cudaStream_t s = as_stream(stream);
  const int64_t tot = (int64_t)k * ncols;
  const int threads = 256;
  const unsigned blocks = (unsigned)((tot + threads - 1) / threads);
  if (y_dtype == SGS_F64)
    return check_ex(launch_ex(partials_reduce_kernel<double>, dim3(blocks), dim3(threads), 0, s,
                              1, partials, nparts, k, ncols, scale, den, static_cast<double*>(Y),
                              ldy, st), "partials_reduce_kernel");
  if (y_dtype == SGS_F32)
    return check_ex(launch_ex(partials_reduce_kernel<float>, dim3(blocks), dim3(threads), 0, s,
                              1, partials, nparts, k, ncols, scale, den, static_cast<float*>(Y),
                              ldy, st), "partials_reduce_kernel");
  set_error("reduce: bad dtype");
  return SGS_EINVAL;
}

extern "C" int sgs_fwht(double* X, int64_t s_len, int ncols, int64_t ldx, void* stream) {
  SGS_REQUIRE(X && s_len >= 1 && ncols >= 1 && ldx >= s_len, "fwht: bad args");
  SGS_REQUIRE((s_len & (s_len - 1)) == 0, "fwht: length %lld is not a power of two",
              (long long)s_len);
  cudaStream_t s = as_stream(stream);
  int L = 0;
  while ((int64_t(1) << L) < s_len) ++L;
  const int lt = L < kSrhtMaxLogT ? L : kSrhtMaxLogT;
  const int64_t ntile = s_len >> lt;
  int rc;
  switch (lt) {
    case 0: return SGS_OK;  // length-1 transform is the identity
    case 1: rc = launch_fwht_tile<1>(X, ldx, ntile, ncols, s); break;
    case 2: rc = launch_fwht_tile<2>(X, ldx, ntile, ncols, s); break;
    case 3: rc = launch_fwht_tile<3>(X, ldx, ntile, ncols, s); break;
    case 4: rc = launch_fwht_tile<4>(X, ldx, ntile, ncols, s); break;
    case 5: rc = launch_fwht_tile<5>(X, ldx, ntile, ncols, s); break;
    case 6: rc = launch_fwht_tile<6>(X, ldx, ntile, ncols, s); break;
    case 7: rc = launch_fwht_tile<7>(X, ldx, ntile, ncols, s); break;
    case 8: rc = launch_fwht_tile<8>(X, ldx, ntile, ncols, s); break;
    case 9: rc = launch_fwht_tile<9>(X, ldx, ntile, ncols, s); break;
    case 10: rc = launch_fwht_tile<10>(X, ldx, ntile, ncols, s); break;
    case 11: rc = launch_fwht_tile<11>(X, ldx, ntile, ncols, s); break;
    default: rc = launch_fwht_tile<12>(X, ldx, ntile, ncols, s); break;
  }
  if (rc) return rc;
  for (int b = lt; b < L; ++b) {
    const int64_t half = s_len >> 1;
    int64_t blocks = (half + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    fwht_global_pass<<<dim3((unsigned)blocks, ncols), 256, 0, s>>>(X, ldx, s_len, int64_t(1) << b);
    rc = check_launch("fwht_global_pass");
    if (rc) return rc;
  }
  return SGS_OK;
}

