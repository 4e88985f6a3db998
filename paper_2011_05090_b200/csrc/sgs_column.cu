// Fused RGS column kernel on sm_100a: the projection update of step 3
// (gram_schmidt.py:316-319) with the P-SRHT sketch of the new column (step 4,
// gram_schmidt.py:320 -> sketch.py:182-184) in its epilogue.
//
// Each CTA owns one 4096-row tile of Q.  It streams Q[:, :i] for its rows with
// evict-first 128-bit loads (8 columns in flight per thread), forms
// q'_i = cast_crs(w) - Q_{i-1} r in registers, stores it, and then - without
// re-reading q' - flips the signs, runs the 4096-point Walsh-Hadamard
// transform (3 bits in registers, 9 bits in three shared-memory radix-8
// passes), gathers the k sampled rows with the cross-tile sign
// (-1)^popcount(r_hi & tile), and sums the k-vectors of its cluster (tile_group CTAs)
// through distributed shared memory.  One partial k-vector per cluster is
// written, exactly as sgs_srht_partials would for a one-tile-per-CTA grid.

#include <cooperative_groups.h>
#include "sgs_common.cuh"
#include "sgs_fwht.cuh"

#include <algorithm>
#include <cstdlib>

namespace cg = cooperative_groups;

namespace sgs {

constexpr int kColThreads = 512;
constexpr int kColLogT = 12;
constexpr int kColT = 1 << kColLogT;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* mb, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mb, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(mb)), "r"(parity) : "memory");
}
// 1-D TMA bulk copy global -> shared with an L2 evict-first hint (the Q stream
// is read once per column and must not evict the reused k-dimensional state).
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* mb, uint64_t policy) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)),
               "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(mb)),
      "l"(policy) : "memory");
}

__device__ __forceinline__ void l2_prefetch(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// L2 prefetch budget (bytes) of the SRHT column kernel's pre-wait prologue:
// about what one LS launch's latency lets HBM move (SGS_COL_PF_MB overrides).
// Issued all at once (one bulk prefetch per thread) the optimum measured at c1
// was 80 MB (48 MB 5777, 64 MB 5820, 80 MB 5841, 96 MB 5807 columns/s): the
// burst of every tile queues up in front of the LS launch's own L2 round trips.
// Paced (col_pf_pace below) a larger budget pays: means of two 20-step runs at
// c1, columns/s - 80 MB burst 5986, 96 MB / 400 cycles 6046, 104 MB / 300-500
// cycles 6045-6054, 112 MB / 400 6035, 120 MB / 800 5814
// (profiles/r02i_prefetch_pacing.txt).  An evict-first policy on the prefetched
// lines changed nothing (6045 vs 6092 without, LS post-wait time the same).  The
// dense ring kernel has its own paced prefetch (launch_dense_ring).
static long col_pf_bytes() {
  static const long b = [] {
    const char* e = getenv("SGS_COL_PF_MB");
    return (e ? atol(e) : 104L) << 20;
  }();
  return b;
}

// Cycles between a tile's successive L2 prefetches (SGS_COL_PF_PACE; 0 = all
// at once, one per thread).
static int col_pf_pace() {
  static const int p = [] {
    const char* e = getenv("SGS_COL_PF_PACE");
    return e ? atoi(e) : 400;
  }();
  return p;
}

// Ring depth: two CTAs per SM (<= 64 registers, __launch_bounds__ below), with
// 4 x 16 KB stages each for fp32 and 3 x 32 KB for fp64.  Two CTAs per SM
// matter for grids of a few waves (c3: 512 tiles): measured at c3 fp64, two
// CTAs x 3 stages 2095 Arnoldi steps/s against one CTA x 6 stages 2024 and
// one CTA x 4 stages 1996.  Large k shrinks the ring to fit shared memory.
template <typename TQ> struct ColCfg;
template <> struct ColCfg<float> { static constexpr int kStages = 4; };
template <> struct ColCfg<double> { static constexpr int kStages = 3; };
constexpr int kColMaxStages = 6;

template <typename TQ>
__host__ __device__ constexpr size_t col_stage_bytes() { return (size_t)kColT * sizeof(TQ); }

template <typename TQ>
__host__ __device__ constexpr size_t col_ring_bytes(int stages) {
  // the FWHT buffer of the epilogue aliases the ring (used after the stream)
  return col_stage_bytes<TQ>() * stages > (size_t)(kColT + kColT / 8 + 8) * 8
             ? col_stage_bytes<TQ>() * stages
             : (size_t)(kColT + kColT / 8 + 8) * 8;
}

// Certification sketch Phi (gram_schmidt.py:333-335) in the same epilogue when
// it is a P-SRHT / block-SRHT with 4096-row tiles: the tile of q' is still in
// registers, so Phi q' costs a second transform and gather, no re-read of q'.
struct ColPhi {
  const uint32_t* sign_bits;  // Phi's sign bitmask, offset to this shard's first row
  const int32_t* samples;     // (nblocks, kphi) block-local sample rows
  int k;
  int log2_block;
  double* partials;           // one kphi-vector per cluster (tile_group tiles)
};

template <typename TQ, typename TW, bool PHI>
__global__ void __launch_bounds__(kColThreads, 2)
rgs_column_kernel(TQ* __restrict__ Q, int64_t ldq, int64_t n, int i,
                  const TW* __restrict__ w, const double* __restrict__ w_div,
                  const TQ* __restrict__ rc, int normalize_prev,
                  const double* __restrict__ R, int64_t ldr, int do_sketch, int64_t row0,
                  int log2_block, const uint32_t* __restrict__ sign_bits,
                  const int32_t* __restrict__ samples, int k, double* __restrict__ partials,
                  const sgs_status* st, unsigned long long* tl, int pf_cols, int nstages,
                  int two, ColPhi phi, int pf_pace, int pf_wave) {
  cg::cluster_group cl = cg::this_cluster();
  if (tl && threadIdx.x == 0) atomicMin(tl + (int64_t)i * 16 + 0, gtimer());
  constexpr int V = VecT<TQ>::N;                  // rows per vector (4 fp32, 2 fp64)
  constexpr int NH = kColT / (kColThreads * V);   // vectors per thread (2 fp32, 4 fp64)
  const int S = nstages;  // ring depth (<= kColMaxStages)
  extern __shared__ __align__(128) unsigned char smem_raw[];
  TQ* ring = reinterpret_cast<TQ*>(smem_raw);                        // S x 4096
  double* z = reinterpret_cast<double*>(smem_raw);                   // aliases the ring
  double* part = reinterpret_cast<double*>(smem_raw + col_ring_bytes<TQ>(S));  // k
  int32_t* smp = reinterpret_cast<int32_t*>(part + k);               // k
  double* part2 = reinterpret_cast<double*>(smp + k + (k & 1));      // PHI: phi.k
  int32_t* smp2 = reinterpret_cast<int32_t*>(part2 + (PHI ? phi.k : 0));  // PHI: phi.k
  TQ* rs = PHI ? reinterpret_cast<TQ*>(smp2 + phi.k + (phi.k & 1))
               : reinterpret_cast<TQ*>(smp + k + (k & 1));           // i coefficients
  __shared__ uint64_t mbar[kColMaxStages];
  // the carve-up (ring | k partials | k samples | [phi] | i coefficients) fits
  SGS_DCHECK(S >= 2 && S <= kColMaxStages && k >= 1);
  SGS_DCHECK(dyn_smem_offset(rs + (i > 0 ? i : 1), smem_raw) <= dyn_smem_bytes());
  SGS_DCHECK(col_ring_bytes<TQ>(S) >= (size_t)(kColT + kColT / 8 + 8) * 8);

  const int tid = threadIdx.x;
  const int64_t lr0 = (int64_t)blockIdx.x * kColT;  // first local row of the tile
  const bool active = lr0 < n;
  const int nvalid = active ? (int)min((int64_t)kColT, n - lr0) : 0;
  const uint32_t bytes = (uint32_t)(((size_t)nvalid * sizeof(TQ) + 15) / 16 * 16);
  const int64_t g0 = row0 + lr0;
  const int64_t blk = g0 >> log2_block;
  const int64_t h = (g0 & ((int64_t(1) << log2_block) - 1)) >> kColLogT;
  const int nplain = (i == 0) ? 0 : (normalize_prev ? i - 1 : i);
  uint64_t policy = 0;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&mbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
  }
  // inputs that do not depend on the predecessor kernel, before waiting on it:
  // the sample rows, this thread's w rows, and the first S columns of Q[:, :i-1]
  if (do_sketch && active) {
    const int32_t* sb = samples + blk * (int64_t)k;
    for (int j = tid; j < k; j += blockDim.x) smp[j] = __ldg(sb + j);
    if constexpr (PHI) {
      const int32_t* sb2 = phi.samples + (g0 >> phi.log2_block) * (int64_t)phi.k;
      for (int j = tid; j < phi.k; j += blockDim.x) smp2[j] = __ldg(sb2 + j);
    }
  }
  __syncthreads();
  // Columns 0..i-2 of Q were finalised by the column kernel before the
  // predecessor (the LS launch, which waited on it before letting this grid
  // start), and w is an input: the ring prologue and the w rows are issued
  // before the dependency wait, so the stream is already in flight when the
  // coefficients r arrive.
  if (tid == 0 && active)
    for (int j = 0; j < S && j < nplain; ++j)
      tma_load_1d(ring + (size_t)j * kColT, Q + (int64_t)j * ldq + lr0, bytes, &mbar[j], policy);
  // The predecessor LS launch keeps HBM idle while it solves: pull the next
  // pf_cols columns of this tile into L2 meanwhile (one bulk prefetch per thread).
  if (pf_pace == 0 && active && tid >= 32 && tid - 32 < pf_cols && S + tid - 32 < nplain)
    l2_prefetch(Q + (int64_t)(S + tid - 32) * ldq + lr0, bytes);
  int64_t rows[NH];
#pragma unroll
  for (int hh = 0; hh < NH; ++hh)
    rows[hh] = lr0 + (int64_t)hh * (kColThreads * V) + (int64_t)tid * V;
  TQ wv[NH][V];
  if (w_div == nullptr) {
#pragma unroll
    for (int hh = 0; hh < NH; ++hh)
#pragma unroll
      for (int v = 0; v < V; ++v)
        wv[hh][v] = (rows[hh] + v < n) ? cvt<TQ>(__ldcs(w + rows[hh] + v)) : TQ(0);
  }
  if (pf_pace > 0 && pf_cols > 0 && (tid >> 5) >= 1 && (tid >> 5) <= 2) {
    // paced variant: warp 1 issues this tile's prefetches one every pf_pace
    // cycles, so the burst of all tiles does not queue up in front of the LS
    // launch's own L2 round trips.  Grids of more than one wave (pf_wave > 0:
    // CTAs below pf_wave are resident before the wait, the others start after
    // it and just stream): warp 2 of a first-wave CTA prefetches for the tile
    // pf_wave further on.
    const bool second = (tid >> 5) == 2;
    const int64_t t = (int64_t)blockIdx.x + (second ? pf_wave : 0);
    const int64_t tr0 = t * kColT;
    bool ok = second ? (pf_wave > 0 && t < (int64_t)gridDim.x && tr0 < n) : active;
    if (pf_wave > 0 && (int)blockIdx.x >= pf_wave) ok = false;
    if (ok) {
      const uint32_t tb =
          (uint32_t)(((size_t)min((int64_t)kColT, n - tr0) * sizeof(TQ) + 15) / 16 * 16);
      const long long t0 = clock64();
      for (int c = 0; c < pf_cols && S + c < nplain; ++c) {
        while (clock64() - t0 < (long long)c * pf_pace) {}
        if ((tid & 31) == (c & 31)) l2_prefetch(Q + (int64_t)(S + c) * ldq + tr0, tb);
      }
    }
  }
  pdl_enter();
  if (w_div != nullptr) {
    // one-synchronisation Arnoldi: w = cast((A q'_{i-1} / alpha) / r_{i-1,i-1}),
    // the divisor finalized by the predecessor launch
    const double d = *w_div;
#pragma unroll
    for (int hh = 0; hh < NH; ++hh)
#pragma unroll
      for (int v = 0; v < V; ++v)
        wv[hh][v] = (rows[hh] + v < n) ? cvt<TQ>((double)__ldcs(w + rows[hh] + v) / d) : TQ(0);
  }
  if (tl && threadIdx.x == 0) atomicMin(tl + (int64_t)i * 16 + 1, gtimer());
  // the first coefficients and the status in one round trip (both are the
  // predecessor LS launch's outputs)
  const TQ rc0 = tid < i ? rc[tid] : TQ(0);
  if (status_stopped(st)) {  // uniform over the grid; drain the prologue before leaving
    if (tid == 0 && active)
      for (int j = 0; j < S && j < nplain; ++j) mbar_wait(&mbar[j], 0u);
    __syncthreads();
    return;
  }
  if (tid < i) rs[tid] = rc0;
  for (int j = tid + blockDim.x; j < i; j += blockDim.x) rs[j] = rc[j];
  __syncthreads();

  // Q_{i-1} r in the coarse dtype, two-level for fp32 (kAccBlock, sgs_common.cuh)
  TQ acc[NH][V], tot[NH][V];
#pragma unroll
  for (int hh = 0; hh < NH; ++hh)
#pragma unroll
    for (int v = 0; v < V; ++v) acc[hh][v] = tot[hh][v] = TQ(0);
  auto fold = [&](int j) {
    if (sizeof(TQ) == 4 && two && ((j + 1) & (kAccBlock - 1)) == 0) {
#pragma unroll
      for (int hh = 0; hh < NH; ++hh)
#pragma unroll
        for (int v = 0; v < V; ++v) {
          tot[hh][v] += acc[hh][v];
          acc[hh][v] = TQ(0);
        }
    }
  };
  if (active) {
    int s = 0;
    uint32_t phase = 0u;  // (j / S) & 1, kept incrementally (S is a runtime depth)
    for (int j = 0; j < nplain; ++j) {
      mbar_wait(&mbar[s], phase);
      const TQ c = rs[j];
      const TQ* buf = ring + (size_t)s * kColT;
#pragma unroll
      for (int hh = 0; hh < NH; ++hh) {
        TQ q[V];
        vload_smem(buf + hh * (kColThreads * V) + tid * V, q);
#pragma unroll
        for (int v = 0; v < V; ++v) acc[hh][v] = fma(q[v], c, acc[hh][v]);
      }
      fold(j);
      __syncthreads();  // everybody has read stage s
      if (tid == 0 && j + S < nplain) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tma_load_1d(ring + (size_t)s * kColT, Q + (int64_t)(j + S) * ldq + lr0, bytes, &mbar[s],
                    policy);
      }
      if (++s == S) {
        s = 0;
        phase ^= 1u;
      }
    }
    if (i > 0 && normalize_prev) {
      const int j = i - 1;
      const double rjj = R[(int64_t)j * ldr + j];
      const TQ c = rs[j];
#pragma unroll
      for (int hh = 0; hh < NH; ++hh) {
        TQ* col = Q + (int64_t)j * ldq + rows[hh];
        if (rows[hh] + V <= n) {
          TQ q[V];
          vload(col, q);
#pragma unroll
          for (int v = 0; v < V; ++v) {
            q[v] = cvt<TQ>((double)q[v] / rjj);
            acc[hh][v] = fma(q[v], c, acc[hh][v]);
          }
          vstore(col, q);
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v)
            if (rows[hh] + v < n) {
              const TQ q = cvt<TQ>((double)col[v] / rjj);
              col[v] = q;
              acc[hh][v] = fma(q, c, acc[hh][v]);
            }
        }
      }
      fold(j);
    }
  }
  double xs[NH * V];  // d o q' of this thread's rows, element order (h, v)
  if (active) {
#pragma unroll
    for (int hh = 0; hh < NH; ++hh) {
      TQ out[V];
#pragma unroll
      for (int v = 0; v < V; ++v)
        out[v] = (rows[hh] + v < n) ? wv[hh][v] - (tot[hh][v] + acc[hh][v]) : TQ(0);
      TQ* dst = Q + (int64_t)i * ldq + rows[hh];
      if (rows[hh] + V <= n) vstore(dst, out);
      else
        for (int v = 0; v < V; ++v)
          if (rows[hh] + v < n) dst[v] = out[v];
      if (do_sketch) {
        const uint32_t word = (rows[hh] < n) ? __ldg(sign_bits + (rows[hh] >> 5)) : 0u;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const double x = (double)out[v];
          const bool pos = (word >> ((rows[hh] + v) & 31)) & 1u;
          xs[hh * V + v] = pos ? x : -x;
        }
      }
    }
  }
  if (!do_sketch) return;  // uniform: no cluster barrier is pending
  // ---- sketch epilogue (z aliases the drained ring) ----------------------------
  __syncthreads();
  if (active) {
    // the stage order of the stand-alone tile kernel (srht_tile_kernel,
    // sgs_sketch.cu): bits 6..11, then 0..5 - four radix-8 passes - so the
    // partials equal sgs_srht_partials' of the same column bit for bit
#pragma unroll
    for (int hh = 0; hh < NH; ++hh)
#pragma unroll
      for (int v = 0; v < V; ++v) z[pidx(hh * (kColThreads * V) + tid * V + v)] = xs[hh * V + v];
    __syncthreads();
#pragma unroll
    for (int b0 : {6, 9, 0, 3}) {
      fwht_pass<kColLogT, 3>(z, b0);
      __syncthreads();
    }
    for (int j = tid; j < k; j += blockDim.x) {
      const int32_t r = smp[j];
      SGS_DCHECK(r >= 0 && (int64_t)r < (int64_t(1) << log2_block));  // block-local sample row
      const double v = z[pidx(r & (kColT - 1))];
      const int64_t rh = (int64_t)(r >> kColLogT);
      part[j] = (__popcll(rh & h) & 1) ? -v : v;
    }
  } else {
    for (int j = tid; j < k; j += blockDim.x) part[j] = 0.0;
  }
  if constexpr (PHI) {
    // Phi q': the same tile from registers with Phi's signs (x = xs * s_theta,
    // so the flip is s_theta XOR s_phi), the same four passes, Phi's samples
    if (active) {
      __syncthreads();  // every thread has gathered Theta's rows from z
      const int64_t hp = (g0 & ((int64_t(1) << phi.log2_block) - 1)) >> kColLogT;
#pragma unroll
      for (int hh = 0; hh < NH; ++hh) {
        const uint32_t wt = (rows[hh] < n) ? __ldg(sign_bits + (rows[hh] >> 5)) : 0u;
        const uint32_t wp = (rows[hh] < n) ? __ldg(phi.sign_bits + (rows[hh] >> 5)) : 0u;
        const uint32_t flip = wt ^ wp;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const double x = xs[hh * V + v];
          z[pidx(hh * (kColThreads * V) + tid * V + v)] =
              ((flip >> ((rows[hh] + v) & 31)) & 1u) ? -x : x;
        }
      }
      __syncthreads();
#pragma unroll
      for (int b0 : {6, 9, 0, 3}) {
        fwht_pass<kColLogT, 3>(z, b0);
        __syncthreads();
      }
      for (int j = tid; j < phi.k; j += blockDim.x) {
        const int32_t r = smp2[j];
        const double v = z[pidx(r & (kColT - 1))];
        const int64_t rh = (int64_t)(r >> kColLogT);
        part2[j] = (__popcll(rh & hp) & 1) ? -v : v;
      }
    } else {
      for (int j = tid; j < phi.k; j += blockDim.x) part2[j] = 0.0;
    }
  }
  cl.sync();
  const int rank = (int)cl.block_rank();
  const int G = (int)cl.num_blocks();  // tile_group(n): tiles per partial
  const int j0 = (int)(((int64_t)rank * k) / G);
  const int j1 = (int)(((int64_t)(rank + 1) * k) / G);
  double* outp = partials + (int64_t)(blockIdx.x / G) * k;
  for (int j = j0 + tid; j < j1; j += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < G; ++q) s += cl.map_shared_rank(part, q)[j];
    outp[j] = s;
  }
  if constexpr (PHI) {
    const int p0 = (int)(((int64_t)rank * phi.k) / G);
    const int p1 = (int)(((int64_t)(rank + 1) * phi.k) / G);
    double* outq = phi.partials + (int64_t)(blockIdx.x / G) * phi.k;
    for (int j = p0 + tid; j < p1; j += blockDim.x) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < G; ++q) s += cl.map_shared_rank(part2, q)[j];
      outq[j] = s;
    }
  }
  cl.sync();
  if (tl && threadIdx.x == 0) atomicMax(tl + (int64_t)i * 16 + 2, gtimer());
}

static int64_t column_ctas(int64_t n_local) {
  const int64_t nt = (n_local + kColT - 1) / kColT;
  const int G = tile_group(n_local);
  return (nt + G - 1) / G * G;
}

// ===========================================================================
// Fused dense-sketch column kernel (Gaussian / Rademacher Theta, step 3 + the
// sketch of step 4 as Theta^T rows): one CTA per row chunk streams, through a
// ring of TMA bulk copies, first the chunk's segments of Q[:, :i] (grouped
// several columns per stage) and then the chunk's rows of Theta^T (contiguous,
// several rows per stage).  q'_i = cast(w) - Q r accumulates per row in column
// order; the GEMV sum_r Theta[:, r] q'_r accumulates per sketch row in row
// order - the chains of the register version.  Chunks are 16-row aligned (the
// bulk copies need 16-byte aligned sources), one partial k-vector per chunk.
constexpr int kDcStageBytes = 53248;  // large bulk copies: measured best (c0)
constexpr int kDcStages = 2;
constexpr int kDcMaxRPT = 4;  // chunk rows per thread

__device__ __forceinline__ void mbar_arrive(uint64_t* mb) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(mb)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* mb, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_copy_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* mb, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(mb)),
      "l"(policy) : "memory");
}

template <typename TQ, typename TW, int QP, bool RAD>
__global__ void __launch_bounds__(512)
dense_ring_kernel(TQ* __restrict__ Q, int64_t ldq, int64_t n, int i, const TW* __restrict__ w,
                  const TQ* __restrict__ rc, int normalize_prev, const double* __restrict__ R,
                  int64_t ldr, int do_sketch, const double* __restrict__ thetaT, int64_t ldt,
                  int k, double* __restrict__ partials, int64_t chunk, int stage_bytes,
                  const sgs_status* st, const uint32_t* __restrict__ rbits, int kw, int two,
                  int pf_stages, int pf_pace) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* ring = smem_raw;  // kDcStages x stage_bytes
  double* xq = reinterpret_cast<double*>(smem_raw + (size_t)kDcStages * stage_bytes);  // chunk
  TQ* rs = reinterpret_cast<TQ*>(xq + chunk);                                           // i
  // full[s]: the stage's bytes landed; empty[s]: every warp has read it
  __shared__ uint64_t full[kDcStages], empty[kDcStages];
  SGS_DCHECK(dyn_smem_offset(rs + (i > 0 ? i : 1), smem_raw) <= dyn_smem_bytes());
  SGS_DCHECK((int64_t)chunk <= (int64_t)kDcMaxRPT * blockDim.x);
  const int tid = threadIdx.x, T = blockDim.x;
  const int nwarps = T >> 5;
  const int p = blockIdx.x;
  const int64_t r0 = (int64_t)p * chunk;
  if (r0 >= n) {  // grid padding (cluster placement): an empty chunk, a zero partial
    pdl_enter();
    if (do_sketch)
      for (int j = threadIdx.x; j < k; j += blockDim.x) partials[(int64_t)p * k + j] = 0.0;
    return;
  }
  const int nr = (int)min(chunk, n - r0);
  const int nplain = (i == 0) ? 0 : (normalize_prev ? i - 1 : i);
  const uint32_t segb = (uint32_t)(((size_t)nr * sizeof(TQ) + 15) / 16 * 16);
  const int G = max(1, stage_bytes / (int)segb);               // Q columns per stage
  const uint32_t rowb = (uint32_t)(ldt * sizeof(double));
  const int Rr = RAD ? 1 : max(1, stage_bytes / (int)rowb);     // Theta rows per stage
  const int n1 = (nplain + G - 1) / G;
  // the Rademacher variant streams only Q through the ring; its +-1 entries
  // come packed (1 bit each, L2-resident) straight from global memory
  const int n2 = (do_sketch && !RAD) ? (nr + Rr - 1) / Rr : 0;
  const int ntot = n1 + n2;
  uint64_t policy = 0;
  if (tid == 0) {
    for (int q = 0; q < kDcStages; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], nwarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
  }
  __syncthreads();
  auto issue = [&](int t) {
    unsigned char* buf = ring + (size_t)(t % kDcStages) * stage_bytes;
    uint64_t* mb = &full[t % kDcStages];
    if (t < n1) {
      const int j0 = t * G, j1 = min(nplain, j0 + G);
      mbar_expect(mb, (uint32_t)(j1 - j0) * segb);
      for (int j = j0; j < j1; ++j)
        tma_copy_1d(buf + (size_t)(j - j0) * segb, Q + (int64_t)j * ldq + r0, segb, mb, policy);
    } else {
      const int rr0 = (t - n1) * Rr, rr1 = min(nr, rr0 + Rr);
      const uint32_t bytes = (uint32_t)(rr1 - rr0) * rowb;
      mbar_expect(mb, bytes);
      tma_copy_1d(buf, thetaT + (r0 + rr0) * ldt, bytes, mb, policy);
    }
  };
  // Q[:, :nplain] and Theta are final before the predecessor started, w is an
  // input: the ring prologue and the w rows go out before the dependency wait
  if (tid == 0)
    for (int t = 0; t < kDcStages && t < ntot; ++t) issue(t);
  TQ wv[kDcMaxRPT];
#pragma unroll
  for (int u = 0; u < kDcMaxRPT; ++u) {
    const int lr = tid + u * T;
    wv[u] = lr < nr ? cvt<TQ>(__ldcs(w + r0 + lr)) : TQ(0);
  }
  // The predecessor LS launch leaves HBM idle: warp 1 pulls the next pf_stages
  // ring stages (the rest of Q[:, :nplain], then this chunk's first rows of
  // Theta^T - the order they are streamed in) into L2, one stage every pf_pace
  // cycles so that the burst does not queue up in front of the LS round trips.
  if (pf_stages > 0 && (tid >> 5) == 1) {
    const int lane = tid & 31;
    const long long t0 = clock64();
    for (int c = 0; c < pf_stages && kDcStages + c < ntot; ++c) {
      const int t = kDcStages + c;
      while (clock64() - t0 < (long long)c * pf_pace) {}
      if (t < n1) {
        const int j0 = t * G, j1 = min(nplain, j0 + G);
        for (int j = j0 + lane; j < j1; j += 32) l2_prefetch(Q + (int64_t)j * ldq + r0, segb);
      } else if (lane == 0) {
        const int rr0 = (t - n1) * Rr, rr1 = min(nr, rr0 + Rr);
        l2_prefetch(thetaT + (r0 + rr0) * ldt, (uint32_t)(rr1 - rr0) * rowb);
      }
    }
  }
  pdl_enter();
  if (status_stopped(st)) {  // uniform; drain the prologue before leaving
    if (tid == 0)
      for (int t = 0; t < kDcStages && t < ntot; ++t) mbar_wait(&full[t], 0u);
    __syncthreads();
    return;
  }
  for (int j = tid; j < i; j += T) rs[j] = rc[j];
  __syncthreads();
  TQ acc[kDcMaxRPT], tot[kDcMaxRPT];  // two-level sum of Q r, as rgs_column_kernel
#pragma unroll
  for (int u = 0; u < kDcMaxRPT; ++u) acc[u] = tot[u] = TQ(0);
  auto fold = [&](int j) {
    if (sizeof(TQ) == 4 && two && ((j + 1) & (kAccBlock - 1)) == 0) {
#pragma unroll
      for (int u = 0; u < kDcMaxRPT; ++u) {
        tot[u] += acc[u];
        acc[u] = TQ(0);
      }
    }
  };
  const int kp = (k + 1) >> 1;
  double2 acc2[QP];
#pragma unroll
  for (int q = 0; q < QP; ++q) acc2[q] = make_double2(0.0, 0.0);
  auto finish_update = [&]() {  // q'_i for the chunk; the Theta stages read xq
#pragma unroll
    for (int u = 0; u < kDcMaxRPT; ++u) {
      const int lr = tid + u * T;
      if (lr >= nr) continue;
      const int64_t r = r0 + lr;
      TQ a = acc[u], tt = tot[u];
      if (i > 0 && normalize_prev) {
        const int jj = i - 1;
        TQ* cp = Q + (int64_t)jj * ldq + r;
        const TQ qn = cvt<TQ>((double)*cp / R[(int64_t)jj * ldr + jj]);
        *cp = qn;
        a = fma(qn, rs[jj], a);
        if (sizeof(TQ) == 4 && two && ((jj + 1) & (kAccBlock - 1)) == 0) {
          tt += a;
          a = TQ(0);
        }
      }
      const TQ out = wv[u] - (tt + a);
      Q[(int64_t)i * ldq + r] = out;
      xq[lr] = (double)out;
    }
    __syncthreads();
  };
  if (n1 == 0) finish_update();
  for (int t = 0; t < ntot; ++t) {
    const int sidx = t % kDcStages;
    const uint32_t ph = (uint32_t)((t / kDcStages) & 1);
    // producer: refill the slot released kDcStages stages ago, as soon as every
    // warp has read it (no block barrier on the consumers' path)
    if (tid == 0 && t >= 1 && t - 1 + kDcStages < ntot) {
      const int tr = t - 1;
      mbar_wait(&empty[tr % kDcStages], (uint32_t)((tr / kDcStages) & 1));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(tr + kDcStages);
    }
    mbar_wait(&full[sidx], ph);
    const unsigned char* buf = ring + (size_t)sidx * stage_bytes;
    if (t < n1) {
      const int j0 = t * G, j1 = min(nplain, j0 + G);
      for (int j = j0; j < j1; ++j) {
        const TQ* col = reinterpret_cast<const TQ*>(buf + (size_t)(j - j0) * segb);
        const TQ c = rs[j];
#pragma unroll
        for (int u = 0; u < kDcMaxRPT; ++u) {
          const int lr = tid + u * T;
          if (lr < nr) acc[u] = fma(col[lr], c, acc[u]);
        }
        fold(j);
      }
    } else {
      const int rr0 = (t - n1) * Rr, rr1 = min(nr, rr0 + Rr);
      for (int rr = rr0; rr < rr1; ++rr) {
        const double xv = xq[rr];
        const double2* trow = reinterpret_cast<const double2*>(buf + (size_t)(rr - rr0) * rowb);
#pragma unroll
        for (int q = 0; q < QP; ++q) {
          const int jj = tid + q * T;
          if (jj < kp) {
            const double2 tv = trow[jj];
            acc2[q].x = fma(tv.x, xv, acc2[q].x);
            acc2[q].y = fma(tv.y, xv, acc2[q].y);
          }
        }
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[sidx]);  // this warp is done with stage t
    if (t == n1 - 1) finish_update();
  }
  if (!do_sketch) return;
  if constexpr (RAD) {
    // Theta q' over the chunk's rows with the device-generated signs: per
    // sketch row the chain in ascending row order, acc + (+-x) - i.e.
    // fma(+-1, x, acc), the materialised Gaussian-path arithmetic exactly
    // (finish_update ended with a block barrier: xq is complete).  U rows of
    // sign words are loaded before they are used, so U L2 round trips are in
    // flight per thread instead of one per row.
    constexpr int U = QP <= 2 ? 16 : (QP <= 4 ? 8 : 4);
    for (int rr0 = 0; rr0 < nr; rr0 += U) {
      uint32_t wd[QP][U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int rr = rr0 + u;
#pragma unroll
        for (int q = 0; q < QP; ++q) {
          const int jj = tid + q * T;
          wd[q][u] = (rr < nr && 2 * jj < k)
                         ? __ldg(rbits + (int64_t)(r0 + rr) * kw + ((2 * jj) >> 5)) : 0u;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int rr = rr0 + u;
        if (rr < nr) {
          const double xv = xq[rr];
#pragma unroll
          for (int q = 0; q < QP; ++q) {
            const int b = (2 * (tid + q * T)) & 31;
            acc2[q].x += ((wd[q][u] >> b) & 1u) ? xv : -xv;
            acc2[q].y += ((wd[q][u] >> (b + 1)) & 1u) ? xv : -xv;
          }
        }
      }
    }
  }
  double* outp = partials + (int64_t)p * k;
#pragma unroll
  for (int q = 0; q < QP; ++q) {
    const int jj = tid + q * T;
    if (2 * jj < k) outp[2 * jj] = acc2[q].x;
    if (2 * jj + 1 < k) outp[2 * jj + 1] = acc2[q].y;
  }
}

// Row chunking of dense_ring_kernel: about two chunks per SM, 16-row aligned,
// at most kDcMaxRPT rows per thread.
// The dense ring grid is chunked for sm_count() - 28 SMs (two CTAs each) and
// launched in clusters of 2 (no DSMEM use: it only makes the placement
// contiguous), so it leaves a GPC free and the column's 16-CTA LS cluster is
// resident from the kernel's start, its pre-wait part overlapping the
// Q/Theta stream (c0: 8632 -> 9045 columns/s; chunking for 104-132 SMs
// measured 8960-9050, for all 148 SMs in clusters of 4 7872).
// SGS_DR_SMS / SGS_DR_CLUSTER override the two choices.
constexpr int kDrReserveSMs = 28;
static int dr_sms() {
  static const int v = [] { const char* e = getenv("SGS_DR_SMS"); return e ? atoi(e) : 0; }();
  return v > 0 ? v : std::max(16, sm_count() - kDrReserveSMs);
}
static int dr_cluster() {
  static const int v = [] { const char* e = getenv("SGS_DR_CLUSTER"); return e ? atoi(e) : 2; }();
  return v > 0 ? v : 1;
}
static void dense_ring_geom(int64_t n, int threads, int64_t* chunk, int* np) {
  int64_t c = (n + 2 * (int64_t)dr_sms() - 1) / (2 * (int64_t)dr_sms());
  const int64_t cmax = (int64_t)kDcMaxRPT * threads / 16 * 16;
  if (c > cmax) c = cmax;
  c = (c + 15) / 16 * 16;
  if (c < 16) c = 16;
  *chunk = c;
  const int cl = dr_cluster();
  *np = (int)(((n + c - 1) / c + cl - 1) / cl * cl);
}

static int dense_ring_threads(int k) {
  const int kp = (k + 1) / 2;
  int threads = ((kp + 31) / 32) * 32;
  if (threads < 256) threads = 256;
  if (threads > 512) threads = 512;
  return threads;
}

template <typename TQ, typename TW, bool RAD>
static int launch_dense_ring(void* Q, int64_t ldq, int64_t n, int i, const void* w,
                             const void* r_crs, int normalize_prev, const double* R, int64_t ldr,
                             int do_sketch, const double* thetaT, int64_t ldt, int k,
                             double* partials, const sgs_status* st, cudaStream_t s,
                             const uint32_t* rbits = nullptr, int kw = 0) {
  const int threads = dense_ring_threads(k);
  const int kp = (k + 1) / 2;
  const int qp = (kp + threads - 1) / threads;
  int64_t chunk;
  int np;
  dense_ring_geom(n, threads, &chunk, &np);
  const int stage_bytes =
      RAD ? kDcStageBytes
          : (int)std::max<int64_t>(kDcStageBytes, ((int64_t)ldt * 8 + 15) / 16 * 16);
  const size_t smem = (size_t)kDcStages * stage_bytes + (size_t)chunk * 8 +
                      (size_t)(i > 0 ? i : 1) * sizeof(TQ);
  if (smem > 227 * 1024) {
    set_error("dense column: k=%d / i=%d need %zu bytes of shared memory", k, i, smem);
    return SGS_EINVAL;
  }
  // pre-wait L2 prefetch (SGS_DENSE_PF_MB total over the grid, 0 = off), paced
  // at the SRHT column kernel's byte rate.  c0, columns/s, two 20-step runs
  // each: off 9123 / 9129, 48 MB 9106 / 9106, 80 MB 9179 / 9166, 104 MB 9168 /
  // 9158, 128 MB 9113 / 9136; the Rademacher variant (Q only) does not move
  // (12 245 at 0, 48 and 104 MB).
  static const long dpf_mb = [] {
    const char* e = getenv("SGS_DENSE_PF_MB");
    return e ? atol(e) : 80L;
  }();
  const int pf_stages = (int)std::min<int64_t>(4096, (dpf_mb << 20) / ((int64_t)np * stage_bytes));
  const int pf_pace = (int)std::min<int64_t>(
      1 << 20, (int64_t)col_pf_pace() * np * stage_bytes / (248 * 16384) + 1);
  cudaError_t e;
#define SGS_DR(QPV)                                                                              \
  do {                                                                                           \
    auto kern = dense_ring_kernel<TQ, TW, QPV, RAD>;                                             \
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);          \
    if (dr_cluster() > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1); \
    e = launch_ex(kern, dim3(np), dim3(threads), smem, s, dr_cluster(), static_cast<TQ*>(Q), ldq, n, i, \
                  static_cast<const TW*>(w), static_cast<const TQ*>(r_crs), normalize_prev, R,   \
                  ldr, do_sketch, thetaT, ldt, k, partials, chunk, stage_bytes, st, rbits, kw,   \
                  acc_two<TQ>(), pf_stages, pf_pace);                                            \
  } while (0)
  if (qp <= 1) SGS_DR(1);
  else if (qp <= 2) SGS_DR(2);
  else if (qp <= 4) SGS_DR(4);
  else if (qp <= 8) SGS_DR(8);
  else {
    set_error("dense column: k=%d too large", k);
    return SGS_EINVAL;
  }
#undef SGS_DR
  return check_ex(e, "dense_ring_kernel");
}

}  // namespace sgs

using namespace sgs;

extern "C" int sgs_dense_column_nparts(int64_t n_local, int k) {
  if (n_local < 1 || k < 1) return 0;
  int64_t chunk;
  int np;
  dense_ring_geom(n_local, dense_ring_threads(k), &chunk, &np);
  return np;
}

extern "C" int sgs_rgs_update_dense(void* Q, int q_dtype, int64_t ldq, int64_t n, int i,
                                    const void* w, int w_dtype, const void* r_crs,
                                    int normalize_prev, const double* R, int64_t ldr,
                                    int do_sketch, const double* thetaT, int64_t ldt, int k,
                                    double* partials, const sgs_status* st, void* stream) {
  SGS_REQUIRE(Q && w && (i == 0 || r_crs) && n >= 1 && i >= 0, "update_dense: bad args");
  SGS_REQUIRE(!normalize_prev || (i > 0 && R), "update_dense: normalize_prev needs R");
  SGS_REQUIRE(!do_sketch || (thetaT && partials && ldt >= k && (ldt % 2) == 0 &&
                             ((uintptr_t)thetaT & 15) == 0), "update_dense: sketch args");
  SGS_REQUIRE(((uintptr_t)Q & 15) == 0 && (ldq % 16) == 0, "update_dense: Q alignment");
  cudaStream_t s = as_stream(stream);
#define SGS_DCL(TQ, TW)                                                                          return launch_dense_ring<TQ, TW, false>(Q, ldq, n, i, w, r_crs, normalize_prev, R, ldr, do_sketch,                                      thetaT, ldt, k, partials, st, s)
  if (q_dtype == SGS_F32 && w_dtype == SGS_F32) SGS_DCL(float, float);
  if (q_dtype == SGS_F32 && w_dtype == SGS_F64) SGS_DCL(float, double);
  if (q_dtype == SGS_F64 && w_dtype == SGS_F32) SGS_DCL(double, float);
  if (q_dtype == SGS_F64 && w_dtype == SGS_F64) SGS_DCL(double, double);
#undef SGS_DCL
  set_error("update_dense: bad dtype");
  return SGS_EINVAL;
}

extern "C" int sgs_rgs_update_rademacher(void* Q, int q_dtype, int64_t ldq, int64_t n, int i,
                                         const void* w, int w_dtype, const void* r_crs,
                                         int normalize_prev, const double* R, int64_t ldr,
                                         int do_sketch, const uint32_t* rbits, int k,
                                         double* partials, const sgs_status* st, void* stream) {
  SGS_REQUIRE(Q && w && (i == 0 || r_crs) && n >= 1 && i >= 0, "update_rademacher: bad args");
  SGS_REQUIRE(!normalize_prev || (i > 0 && R), "update_rademacher: normalize_prev needs R");
  SGS_REQUIRE(!do_sketch || (rbits && partials && k >= 1), "update_rademacher: sketch args");
  SGS_REQUIRE(((uintptr_t)Q & 15) == 0 && (ldq % 16) == 0, "update_rademacher: Q alignment");
  cudaStream_t s = as_stream(stream);
  const int kw = (k + 31) / 32;
#define SGS_RCL(TQ, TW)                                                                        \
  return launch_dense_ring<TQ, TW, true>(Q, ldq, n, i, w, r_crs, normalize_prev, R, ldr,       \
                                         do_sketch, nullptr, 0, k, partials, st, s, rbits, kw)
  if (q_dtype == SGS_F32 && w_dtype == SGS_F32) SGS_RCL(float, float);
  if (q_dtype == SGS_F32 && w_dtype == SGS_F64) SGS_RCL(float, double);
  if (q_dtype == SGS_F64 && w_dtype == SGS_F32) SGS_RCL(double, float);
  if (q_dtype == SGS_F64 && w_dtype == SGS_F64) SGS_RCL(double, double);
#undef SGS_RCL
  set_error("update_rademacher: bad dtype");
  return SGS_EINVAL;
}

extern "C" int sgs_column_nparts(int64_t n_local) {
  return n_local < 1 ? 0 : (int)(column_ctas(n_local) / tile_group(n_local));
}

static int update_srht_impl(void* Q, int q_dtype, int64_t ldq, int64_t n, int i, const void* w,
                             int w_dtype, const double* w_div, const void* r_crs,
                             int normalize_prev, const double* R, int64_t ldr, int do_sketch,
                             int64_t row0, int log2_block, const uint32_t* sign_bits,
                             const int32_t* samples, int k, double* partials,
                             const uint32_t* phi_sign_bits, const int32_t* phi_samples, int kphi,
                             int phi_log2_block, double* phi_partials,
                             const sgs_status* st, void* stream) {
  SGS_REQUIRE(Q && w, "update_srht: null pointer");
  const bool use_phi = phi_partials != nullptr;
  SGS_REQUIRE(!use_phi || (do_sketch && phi_sign_bits && phi_samples && kphi >= 1 &&
                           kphi <= 8192 && phi_log2_block >= kColLogT),
              "update_srht: certification sketch arguments (P-SRHT, 4096-row tiles)");
  SGS_REQUIRE(i >= 0 && n >= 1 && ldq >= n && (ldq % 4) == 0, "update_srht: bad sizes");
  SGS_REQUIRE(i == 0 || r_crs, "update_srht: r_crs required for i > 0");
  SGS_REQUIRE(!normalize_prev || (i > 0 && R), "update_srht: normalize_prev needs R, i > 0");
  SGS_REQUIRE(((uintptr_t)Q & 15) == 0, "update_srht: Q must be 16-byte aligned");
  SGS_REQUIRE(!do_sketch || (sign_bits && samples && partials && k >= 1 && k <= 8192),
              "update_srht: sketch arguments");
  SGS_REQUIRE(!do_sketch || (log2_block >= kColLogT && (row0 % kColT) == 0),
              "update_srht: needs 4096-row tiles (log2_block >= 12, row0 %% 4096 == 0)");
  cudaStream_t s = as_stream(stream);
  const int64_t nctas = column_ctas(n);
  const int esz = q_dtype == SGS_F32 ? 4 : 8;
  const size_t rest = (size_t)k * sizeof(double) + (size_t)(k + 1) * sizeof(int32_t) + 8 +
                      (use_phi ? (size_t)kphi * sizeof(double) + (size_t)(kphi + 1) * 4 : 0) +
                      (size_t)(i > 0 ? i : 1) * esz;
  int nst = q_dtype == SGS_F32 ? ColCfg<float>::kStages : ColCfg<double>::kStages;
  auto ring_of = [&](int st_) {
    return q_dtype == SGS_F32 ? col_ring_bytes<float>(st_) : col_ring_bytes<double>(st_);
  };
  {
    static int env_st = -1;  // SGS_COL_STAGES: experiment override of the ring depth
    if (env_st < 0) {
      const char* e = getenv("SGS_COL_STAGES");
      env_st = e ? std::max(2, std::min(kColMaxStages, atoi(e))) : 0;
    }
    if (env_st > 0) nst = env_st;
  }
  while (nst > 2 && ring_of(nst) + rest > 227 * 1024) --nst;  // large k / i: shallower ring
  const size_t smem = ring_of(nst) + rest;
  SGS_REQUIRE(smem <= 227 * 1024, "update_srht: i=%d k=%d needs %zu bytes of shared memory", i,
              k, smem);
  // L2 prefetch of the columns behind the ring prologue, spread over the tiles.
  // A grid of one wave prefetches per tile; a larger one (c3: 512 tiles) only
  // with the paced variant, whose first-wave CTAs (taken as 2 per SM on the SMs
  // the LS cluster leaves free) also cover the tiles of the next wave.  The
  // pace is scaled so that the whole grid issues bytes at c1's rate.
  // Measured at c3 (512 tiles; Arnoldi steps/s with / without): f64 2078 / 2001,
  // fp32 basis 3443 / 3496, one-sync 2138 / 2152 and 3620 / 3751 - no gain, so
  // multi-wave grids prefetch only with SGS_COL_PF_MULTI=1.
  static const bool pf_multi = [] {
    const char* e = getenv("SGS_COL_PF_MULTI");
    return e && atoi(e) != 0;
  }();
  const int pace0 = col_pf_pace();
  const int64_t wave = 2 * (148 - 16);
  const bool multi = nctas > 2 * 148;
  int pf = (multi && (!pf_multi || pace0 == 0 || nctas > 2 * wave))
               ? 0
               : (int)std::min<int64_t>(kColThreads - 32, col_pf_bytes() / (nctas * kColT * esz));
  const int pf_wave = multi ? (int)wave : 0;
  const int pace = (int)std::min<int64_t>(
      1 << 20, (int64_t)pace0 * nctas * esz / (248 * 4) + (pace0 > 0 ? 1 : 0));
  cudaError_t err = cudaSuccess;
  const ColPhi phi{phi_sign_bits, phi_samples, use_phi ? kphi : 0, phi_log2_block, phi_partials};
#define SGS_COL(TQ, TW)                                                                       \
  do {                                                                                        \
    auto kern = use_phi ? rgs_column_kernel<TQ, TW, true> : rgs_column_kernel<TQ, TW, false>; \
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);       \
    err = launch_ex(kern, dim3((unsigned)nctas), dim3(kColThreads), smem, s, tile_group(n),   \
                    static_cast<TQ*>(Q), ldq, n, i, static_cast<const TW*>(w), w_div,        \
                    static_cast<const TQ*>(r_crs), normalize_prev, R, ldr, do_sketch, row0,  \
                    log2_block, sign_bits, samples, k, partials, st, debug_timeline(), pf,    \
                    nst, acc_two<TQ>(), phi, pace, pf_wave);                                  \
  } while (0)
  if (q_dtype == SGS_F32 && w_dtype == SGS_F32) SGS_COL(float, float);
  else if (q_dtype == SGS_F32 && w_dtype == SGS_F64) SGS_COL(float, double);
  else if (q_dtype == SGS_F64 && w_dtype == SGS_F32) SGS_COL(double, float);
  else if (q_dtype == SGS_F64 && w_dtype == SGS_F64) SGS_COL(double, double);
  else {
    set_error("update_srht: bad dtype");
    return SGS_EINVAL;
  }
#undef SGS_COL
  return check_ex(err, "rgs_column_kernel");
}

extern "C" int sgs_rgs_update_srht_phi(void* Q, int q_dtype, int64_t ldq, int64_t n, int i,
                                       const void* w, int w_dtype, const double* w_div,
                                       const void* r_crs, int normalize_prev, const double* R,
                                       int64_t ldr, int do_sketch, int64_t row0, int log2_block,
                                       const uint32_t* sign_bits, const int32_t* samples, int k,
                                       double* partials, const uint32_t* phi_sign_bits,
                                       const int32_t* phi_samples, int kphi, int phi_log2_block,
                                       double* phi_partials, const sgs_status* st,
                                       void* stream) {
  return update_srht_impl(Q, q_dtype, ldq, n, i, w, w_dtype, w_div, r_crs, normalize_prev, R, ldr,
                          do_sketch, row0, log2_block, sign_bits, samples, k, partials,
                          phi_sign_bits, phi_samples, kphi, phi_log2_block, phi_partials, st,
                          stream);
}

extern "C" int sgs_rgs_update_srht(void* Q, int q_dtype, int64_t ldq, int64_t n, int i,
                                   const void* w, int w_dtype, const double* w_div,
                                   const void* r_crs, int normalize_prev, const double* R,
                                   int64_t ldr, int do_sketch, int64_t row0, int log2_block,
                                   const uint32_t* sign_bits, const int32_t* samples, int k,
                                   double* partials, const sgs_status* st, void* stream) {
  return sgs_rgs_update_srht_phi(Q, q_dtype, ldq, n, i, w, w_dtype, w_div, r_crs, normalize_prev,
                                 R, ldr, do_sketch, row0, log2_block, sign_bits, samples, k,
                                 partials, nullptr, nullptr, 0, 0, nullptr, st, stream);
}
