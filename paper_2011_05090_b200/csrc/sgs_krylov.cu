// RGMRES support kernels on sm_100a: CSR SpMV with the gmres 1/alpha scaling
// (krylov.py:81-83, :276), deterministic norms, the power-iteration step of
// _operator_norm_estimate (krylov.py:213-226) and the progressive Givens
// update (krylov.py:282-301) so the Arnoldi loop never waits on the host.

#include <cstdlib>
#include "sgs_common.cuh"
#include "sgs_fwht.cuh"

namespace sgs {

std::atomic<uint64_t> g_launches{0};

static thread_local char g_err[512] = {0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static unsigned long long* g_timeline = nullptr;
static int64_t g_timeline_col = 0;
unsigned long long* debug_timeline() { return g_timeline; }
unsigned long long* debug_timeline_row() {
  return g_timeline ? g_timeline + g_timeline_col * 16 : nullptr;
}

bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SGS_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

bool acc_two_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SGS_ACC_TWO");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

int sm_count() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached = v > 0 ? v : kMaxSMs;
  }
  return cached;
}

// y = (A x) / alpha with, when xdiv != NULL, x = cast(q / xdiv[0]) formed on the
// fly from a not yet normalised basis column (the rounding the next column
// kernel applies when it normalises q in place).
// Staged CSR SpMV: one CTA per kSpRows consecutive rows.  Their nonzeros are
// contiguous, so one elected thread copies the CTA's column indices and values
// into shared memory with two TMA bulk copies (evict-first: the CSR stream is
// read once per step and must not push x or the sketch state out of L2), issued
// BEFORE the dependency wait - the matrix does not depend on the predecessor,
// so resident CTAs stream it while the previous kernel drains.  Then thread per
// row, one fma chain per row in storage order, reading the row's entries from
// shared memory instead of strided global loads.  A CTA whose
// range exceeds the buffer, or whose 16-byte-rounded copy would run past the
// arrays' end, takes the global path (same arithmetic).
constexpr int kSpRows = 512;
constexpr int kSpThreads = 256;
constexpr int kSpCap = kSpRows * 7 + 8;  // staged entries per CTA (7-point stencils fit)

__device__ __forceinline__ uint32_t sp_smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

template <typename TX>
__device__ __forceinline__ double sp_xval(const TX* __restrict__ x, int c, const double* xdiv,
                                          double dv) {
  const TX xr = __ldg(x + c);
  if (xdiv == nullptr) return (double)xr;
  if constexpr (sizeof(TX) == 4) return (double)__double2float_rn((double)xr / dv);
  else return (double)xr / dv;
}

// The rows of one CTA (kSpRows) of y = (A x) / alpha, staged through svals /
// sci / mbar (shared memory).  Returns true when the status block stopped the
// launch (nothing written).
template <typename TX>
__device__ __forceinline__ bool spmv_block(int64_t n, const int32_t* __restrict__ rp,
                                           const int32_t* __restrict__ ci,
                                           const double* __restrict__ vals,
                                           const TX* __restrict__ x,
                                           const double* __restrict__ xdiv,
                                           const double* __restrict__ alpha,
                                           double* __restrict__ y, const sgs_status* st,
                                           unsigned long long* tl, int allow_stage,
                                           double* svals, int32_t* sci, uint64_t* mbar) {
  const int64_t r0 = (int64_t)blockIdx.x * kSpRows;
  const int64_t r1 = min(n, r0 + kSpRows);
  const int b = __ldg(rp + r0), e = __ldg(rp + r1), nnz = __ldg(rp + n);
  // 16-byte aligned source ranges covering [b, e)
  const int b_ci = b & ~3, e_ci = (e + 3) & ~3;
  const int b_v = b & ~1, e_v = (e + 1) & ~1;
  const bool staged = allow_stage && (e_ci - b_ci) <= kSpCap + 4 && (e_v - b_v) <= kSpCap + 2 &&
                      e_ci <= nnz && e_v <= nnz && e > b;
  SGS_DCHECK(b >= 0 && b <= e && e <= nnz);
  int rb[2], re[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t r = r0 + threadIdx.x + h * kSpThreads;
    rb[h] = r < r1 ? __ldg(rp + r) : 0;
    re[h] = r < r1 ? __ldg(rp + r + 1) : 0;
  }
  if (staged && threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sp_smem_u32(mbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const uint32_t bci = (uint32_t)(e_ci - b_ci) * 4u, bv = (uint32_t)(e_v - b_v) * 8u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sp_smem_u32(mbar)),
                 "r"(bci + bv) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(sp_smem_u32(sci)), "l"(ci + b_ci), "r"(bci),
        "r"(sp_smem_u32(mbar)), "l"(pol) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(sp_smem_u32(svals)), "l"(vals + b_v), "r"(bv),
        "r"(sp_smem_u32(mbar)), "l"(pol) : "memory");
  }
  __syncthreads();
  pdl_enter();
  if (tl && threadIdx.x == 0) atomicMin(tl + 9, gtimer());
  if (status_stopped(st)) {
    if (staged) {  // drain the copies before the shared memory goes away
      asm volatile(
          "{\n\t.reg .pred p;\nW0_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
          "@!p bra W0_%=;\n}" ::"r"(sp_smem_u32(mbar)) : "memory");
    }
    return true;
  }
  const double dv = xdiv ? __ldg(xdiv) : 1.0;
  const double ia = alpha ? __ldg(alpha) : 1.0;
  if (staged) {
    asm volatile(
        "{\n\t.reg .pred p;\nW1_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
        "@!p bra W1_%=;\n}" ::"r"(sp_smem_u32(mbar)) : "memory");
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t r = r0 + threadIdx.x + h * kSpThreads;
    if (r >= r1) continue;
    double acc = 0.0;
    if (staged) {
      const int32_t* pc = sci + (rb[h] - b_ci);
      const double* pv = svals + (rb[h] - b_v);
      const int len = re[h] - rb[h];
#pragma unroll 8
      for (int q = 0; q < len; ++q) acc = fma(pv[q], sp_xval(x, pc[q], xdiv, dv), acc);
    } else {
      for (int q = rb[h]; q < re[h]; ++q) acc = fma(__ldg(vals + q), sp_xval(x, __ldg(ci + q), xdiv, dv), acc);
    }
    y[r] = alpha ? acc / ia : acc;
  }
  if (tl) {
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(tl + 10, gtimer());
  }
  return false;
}

template <typename TX>
__global__ void __launch_bounds__(kSpThreads)
csr_spmv_staged_kernel(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                       const double* __restrict__ vals, const TX* __restrict__ x,
                       const double* __restrict__ xdiv, const double* __restrict__ alpha,
                       double* __restrict__ y, const sgs_status* st, unsigned long long* tl,
                       int allow_stage) {
  __shared__ __align__(16) double svals[kSpCap + 2];
  __shared__ __align__(16) int32_t sci[kSpCap + 4];
  __shared__ __align__(8) uint64_t mbar;
  spmv_block<TX>(n, rp, ci, vals, x, xdiv, alpha, y, st, tl, allow_stage, svals, sci, &mbar);
}

// ---------------------------------------------------------------------------
// SpMV with the SRHT of its output fused in (RGMRES's w = A q and p = Theta w,
// one launch instead of two and no HBM re-read of w).  The CTAs are the plain
// staged SpMV's (kSpRows rows each, kSpPerTile per 4096-row SRHT tile).  A CTA
// publishes its rows of w (barrier, one device-scope fence, a per-tile
// counter); the CTA that completes a tile transforms it from L2 with the
// 256-thread three-phase register FWHT of srht_tile3_kernel (levels 6..9 |
// 10, 11, 0, 1 | 2..5, the level order of every SRHT kernel here), gathers
// the tile's k sampled rows into a tile vector (0.0 + (+-z), as one tile of
// the clustered tile kernel) and bumps a per-group counter; the CTA that
// completes a group of tile_group(n) tiles sums their tile vectors in tile
// order from 0.0 - the DSMEM cluster sum of srht_tile_kernel - into the
// group's partial.  So the partials are the stand-alone sketch's bit for bit.
// The counters are monotonic (every CTA counts, also when the status block
// stopped the launch), so they never need a reset.
constexpr int kSpTile = 4096;
constexpr int kSpPerTile = kSpTile / kSpRows;  // CTAs per SRHT tile
constexpr int kSpT3Buf = 4096 + 256;           // padded tile: slot e + e / 16
__device__ __forceinline__ int sp_t3idx(int e) { return e + (e >> 4); }

struct SpmvSrht {
  int64_t row0;               // global row of local row 0 (shard offset)
  int log2_block;             // SRHT block (>= 12)
  const uint32_t* sign_bits;  // sign word of local rows 32 w .. 32 w + 31 at [w]
  const int32_t* samples;     // k sample rows per block
  int k;
  int G;                      // tiles per partial: tile_group(n)
  double* tilevec;            // ntiles x k scratch
  unsigned long long* counters;  // ntiles tile counters, then ngroups group counters
  double* partials;           // ngroups x k
};

template <typename TX, int KQ>
__global__ void __launch_bounds__(kSpThreads, 5)  // 5 CTAs per SM, as the plain SpMV
csr_spmv_srht_kernel(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                     const double* __restrict__ vals, const TX* __restrict__ x,
                     const double* __restrict__ xdiv, const double* __restrict__ alpha,
                     double* __restrict__ y, const sgs_status* st, unsigned long long* tl,
                     int allow_stage, SpmvSrht sk) {
  extern __shared__ __align__(16) unsigned char sp_dyn[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ int s_last;
  double* svals = reinterpret_cast<double*>(sp_dyn);
  int32_t* sci = reinterpret_cast<int32_t*>(sp_dyn + (size_t)(kSpCap + 2) * 8);
  const bool stop = spmv_block<TX>(n, rp, ci, vals, x, xdiv, alpha, y, st, tl, allow_stage,
                                   svals, sci, &mbar);
  const int t = threadIdx.x;
  const int64_t tile = (int64_t)blockIdx.x / kSpPerTile;
  const int64_t ntiles = (n + kSpTile - 1) / kSpTile;
  const int64_t lr0 = tile * kSpTile;
  // ---- tile completion: this CTA's rows of w are published
  __syncthreads();  // every row of the CTA stored; the staging buffers are free
  if (t == 0) {
    __threadfence();
    const unsigned long long per =
        (unsigned long long)((min(n, lr0 + kSpTile) - lr0 + kSpRows - 1) / kSpRows);
    const unsigned long long old = atomicAdd(sk.counters + tile, 1ull);
    s_last = ((old + 1) % per) == 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();  // the other CTAs' rows of this tile
  if (tl && t == 0) atomicMin(tl + 12, gtimer());
  // shared memory reused: the padded tile, 128 sign words, the k samples
  double* buf = svals;
  uint32_t* sgn = reinterpret_cast<uint32_t*>(sp_dyn + (size_t)kSpT3Buf * 8);
  int32_t* smp = reinterpret_cast<int32_t*>(sgn + 128);
  SGS_DCHECK(dyn_smem_offset(smp + sk.k, sp_dyn) <= dyn_smem_bytes());
  if (!stop) {
    constexpr int LOGT = 12;
    const int64_t g0 = sk.row0 + lr0;
    const int64_t blk = g0 >> sk.log2_block;
    const int64_t h = (g0 & ((int64_t(1) << sk.log2_block) - 1)) >> LOGT;
    const int ea = (t & 63) | ((t >> 6) << 10);
    double v[16];
    if (lr0 + kSpTile <= n) {
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = __ldcg(y + lr0 + ea + 64 * r);
    } else {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int64_t lr = lr0 + ea + 64 * r;
        v[r] = lr < n ? __ldcg(y + lr) : 0.0;
      }
    }
    if (t < kSpTile / 32)
      sgn[t] = (lr0 + 32 * (int64_t)t < n) ? __ldg(sk.sign_bits + (lr0 >> 5) + t) : ~0u;
    const int32_t* sb = sk.samples + blk * (int64_t)sk.k;
    for (int j = t; j < sk.k; j += kSpThreads) smp[j] = __ldg(sb + j);
    __syncthreads();
    const uint32_t* sgw = sgn + (ea >> 5);
#pragma unroll
    for (int r = 0; r < 16; ++r)
      if (((sgw[2 * r] >> (t & 31)) & 1u) == 0u) v[r] = -v[r];
    fwht_reg<4>(v);  // bits 6..9
    double* const pa = buf + sp_t3idx(ea);
#pragma unroll
    for (int r = 0; r < 16; ++r) pa[68 * r] = v[r];
    __syncthreads();
    double* const pb = buf + sp_t3idx(t << 2);
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = pb[(r >> 2) + 1088 * (r & 3)];
    fwht_reg<4>(v);  // bits 10, 11, 0, 1
#pragma unroll
    for (int r = 0; r < 16; ++r) pb[(r >> 2) + 1088 * (r & 3)] = v[r];
    __syncthreads();
    double* const pc = buf + sp_t3idx((t & 3) | ((t >> 2) << 6));
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = pc[4 * r + (r >> 2)];
    fwht_reg<4>(v);  // bits 2..5
#pragma unroll
    for (int r = 0; r < 16; ++r) pc[4 * r + (r >> 2)] = v[r];
    __syncthreads();
    double* tv = sk.tilevec + tile * (int64_t)sk.k;
#pragma unroll
    for (int q = 0; q < KQ; ++q) {
      const int j = t + kSpThreads * q;
      if (j < sk.k) {
        const int32_t r = smp[j];
        SGS_DCHECK(r >= 0 && (int64_t)r < (int64_t(1) << sk.log2_block));
        const double z = buf[sp_t3idx(r & (kSpTile - 1))];
        const int64_t rh = (int64_t)(r >> LOGT);
        tv[j] = 0.0 + ((__popcll(rh & h) & 1) ? -z : z);
      }
    }
  }
  // ---- group completion
  __syncthreads();
  const int64_t grp = tile / sk.G;
  const int64_t ngroups = (ntiles + sk.G - 1) / sk.G;
  if (t == 0) {
    __threadfence();
    const unsigned long long per = (unsigned long long)min((int64_t)sk.G, ntiles - grp * sk.G);
    const unsigned long long old = atomicAdd(sk.counters + ntiles + grp, 1ull);
    s_last = ((old + 1) % per) == 0;
  }
  __syncthreads();
  if (!s_last || stop) return;
  __threadfence();
  const int64_t gt0 = grp * sk.G;
  const int nt = (int)min((int64_t)sk.G, ntiles - gt0);
  double* out = sk.partials + grp * (int64_t)sk.k;
  for (int j = t; j < sk.k; j += kSpThreads) {
    double acc = 0.0;
    for (int q = 0; q < nt; ++q) acc += __ldcg(sk.tilevec + (gt0 + q) * (int64_t)sk.k + j);
    out[j] = acc;
  }
  (void)ngroups;
  if (tl) {
    __syncthreads();
    if (t == 0) atomicMax(tl + 13, gtimer());
  }
}

constexpr int kNormBlocks = 296;

template <typename TX>
__global__ void __launch_bounds__(256)
norm_partial_kernel(const TX* __restrict__ x, int64_t n, double* __restrict__ work) {
  __shared__ double red[8];
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t b = per * blockIdx.x, e = min(n, b + per);
  double acc = 0.0;
  for (int64_t r = b + threadIdx.x; r < e; r += blockDim.x) {
    const double v = (double)x[r];
    acc = fma(v, v, acc);
  }
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) work[blockIdx.x] = s;
}

__global__ void norm_final_kernel(const double* __restrict__ work, int nb, double* out) {
  __shared__ double red[8];
  double acc = 0.0;
  for (int q = threadIdx.x; q < nb; q += blockDim.x) acc += work[q];
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) out[0] = sqrt(s);
}

__global__ void scale_kernel(const double* __restrict__ x, double num, const double* den,
                             int divide, double* __restrict__ y, int64_t n) {
  double f;
  if (divide) f = *den;
  else f = den ? num / *den : num;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    y[r] = divide ? x[r] / f : f * x[r];
}

__global__ void rsub_kernel(const double* __restrict__ b, double* __restrict__ y, int64_t n) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    y[r] = b[r] - y[r];
}

template <typename TS, typename TD>
__global__ void cast_div_kernel(const TS* __restrict__ x, const double* den, TD* __restrict__ y,
                                int64_t n) {
  const double d = den ? *den : 1.0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const double v = den ? (double)x[r] / d : (double)x[r];
    y[r] = from_double<TD>(v);
  }
}

__global__ void power_step_kernel(const double* __restrict__ w, const double* nrm,
                                  double* __restrict__ v, double* sigma, int64_t n) {
  const double nw = *nrm;
  // sigma < 0 marks "frozen": a zero norm was seen, estimate is 0 (krylov.py:220-221)
  if (*sigma < 0.0) return;
  if (nw == 0.0) {
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) *sigma = -1.0;
    return;
  }
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    v[r] = w[r] / nw;
}

__global__ void power_commit_kernel(const double* nrm, double* sigma) {
  if (*sigma < 0.0) return;
  if (*nrm != 0.0) *sigma = *nrm;
}

__global__ void cos_init_kernel(double* v, int64_t n, int64_t first) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    v[r] = cos((double)(first + r) + 1.0);
}

// One progressive Givens step (krylov.py:282-301).  The O(i) rotation chain
// is sequential; the Hessenberg column and the rotations are staged in shared
// memory by the whole block so the single-thread chain only touches shared
// memory.  Products and sums are not contracted so the arithmetic matches
// numpy's scalar expressions.
constexpr int kGivMax = 4096;
// One progressive Givens update by the calling block (all its threads).
__device__ __forceinline__ void givens_update(const double* __restrict__ R, int64_t ldr, int i,
                                              double* cs, double* sn, double* g, double* T,
                                              int64_t ldt, double* hist, double tol,
                                              sgs_status* st, unsigned long long* tl) {
  extern __shared__ double gsm[];
  double* h = gsm;            // i + 2
  double* c_s = gsm + i + 2;  // i
  double* s_s = c_s + i;      // i
  const double* rc = R + (int64_t)(i + 1) * ldr;
  for (int j = threadIdx.x; j < i + 2; j += blockDim.x) h[j] = rc[j];
  for (int j = threadIdx.x; j < i; j += blockDim.x) {
    c_s[j] = cs[j];
    s_s[j] = sn[j];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double beta = R[0];
    if (i == 0) g[0] = beta;
    double carry = h[0];
    // the dependent chain runs from registers: 8 rotations and h entries are
    // loaded one chunk ahead (a chunk writes h[j..j+7] and the next reads
    // h[j+9..j+16]), so no shared-memory latency sits on the carry
    constexpr int kU = 8;
    const int nfull = i / kU * kU;
    double cc[kU], ss[kU], hh[kU];
    if (nfull > 0) {
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        cc[u] = c_s[u];
        ss[u] = s_s[u];
        hh[u] = h[u + 1];
      }
    }
    for (int j = 0; j < nfull; j += kU) {
      double nc[kU], ns[kU], nh[kU], ho[kU];
      const bool more = j + kU < nfull;
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        nc[u] = more ? c_s[j + kU + u] : 0.0;
        ns[u] = more ? s_s[j + kU + u] : 0.0;
        nh[u] = more ? h[j + kU + u + 1] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        ho[u] = __dadd_rn(__dmul_rn(cc[u], carry), __dmul_rn(ss[u], hh[u]));
        carry = __dadd_rn(__dmul_rn(-ss[u], carry), __dmul_rn(cc[u], hh[u]));
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        h[j + u] = ho[u];
        cc[u] = nc[u];
        ss[u] = ns[u];
        hh[u] = nh[u];
      }
    }
    for (int j = nfull; j < i; ++j) {
      const double c = c_s[j], s = s_s[j], hn = h[j + 1];
      h[j] = __dadd_rn(__dmul_rn(c, carry), __dmul_rn(s, hn));
      carry = __dadd_rn(__dmul_rn(-s, carry), __dmul_rn(c, hn));
    }
    h[i] = carry;
    const double r = hypot(h[i], h[i + 1]);
    double c, s;
    if (r == 0.0) { c = 1.0; s = 0.0; }
    else { c = h[i] / r; s = h[i + 1] / r; }
    cs[i] = c;
    sn[i] = s;
    h[i] = r;
    h[i + 1] = 0.0;
    const double gi = g[i];
    g[i + 1] = __dmul_rn(-s, gi);
    g[i] = __dmul_rn(c, gi);
    const double est = fabs(g[i + 1]) / beta;
    hist[i] = est;
    st->iters = i + 1;
    if (tol >= 0.0 && est <= tol) {
      st->code = SGS_ST_CONVERGED;
      st->column = i + 1;
    }
  }
  __syncthreads();
  double* Tc = T + (int64_t)i * ldt;
  for (int j = threadIdx.x; j < i + 2; j += blockDim.x) Tc[j] = h[j];
  if (tl && threadIdx.x == 0) tl[(int64_t)(i + 1) * 16 + 11] = gtimer();
}

__global__ void __launch_bounds__(256)
givens_step_kernel(const double* __restrict__ R, int64_t ldr, int i, double* cs, double* sn,
                   double* g, double* T, int64_t ldt, double* hist, double tol, sgs_status* st,
                   unsigned long long* tl) {
  pdl_enter();
  if (status_stopped(st)) return;
  givens_update(R, ldr, i, cs, sn, g, T, ldt, hist, tol, st, tl);
}

constexpr int kHeadPer = 4;
// Head of an RGMRES step: the last block performs the Givens update of step
// gi (if gi >= 0) while all other blocks normalise basis column `col` in
// place.  The normalising blocks ignore the status block on purpose - the
// Givens update may set CONVERGED concurrently, and a partly normalised
// column must never happen; *norm_flag = col records what was normalised.
template <typename TQ>
__global__ void __launch_bounds__(256)
arnoldi_head_kernel(TQ* __restrict__ Q, int64_t ldq, int64_t n, int col, int* norm_flag, int gi,
                    const double* __restrict__ R, int64_t ldr, double* cs, double* sn, double* g,
                    double* T, int64_t ldt, double* hist, double tol, sgs_status* st,
                    unsigned long long* tl) {
  pdl_enter();
  if (gi >= 0 && blockIdx.x == gridDim.x - 1) {
    if (!status_stopped(st)) givens_update(R, ldr, gi, cs, sn, g, T, ldt, hist, tol, st, tl);
    return;
  }
  if (col < 0) return;
  const double rjj = R[(int64_t)col * ldr + col];
  TQ* q = Q + (int64_t)col * ldq;
  // kHeadPer elements per thread, all loads issued before the divisions (a
  // grid-stride loop here waits one memory latency per element)
  const int64_t r0 = (int64_t)blockIdx.x * blockDim.x * kHeadPer + threadIdx.x;
  TQ v[kHeadPer];
#pragma unroll
  for (int u = 0; u < kHeadPer; ++u) {
    const int64_t r = r0 + (int64_t)u * blockDim.x;
    v[u] = r < n ? q[r] : TQ(0);
  }
#pragma unroll
  for (int u = 0; u < kHeadPer; ++u) {
    const int64_t r = r0 + (int64_t)u * blockDim.x;
    if (r < n) q[r] = cvt<TQ>((double)v[u] / rjj);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *norm_flag = col;
}


__global__ void status_init_kernel(sgs_status* st) {
  st->code = 0;
  st->column = 0;
  st->ncols = 0;
  st->iters = 0;
  st->r_ii = 0.0;
  st->tol = 0.0;
  st->diag_max = 0.0;
  st->diag_min = 0.0;
}

static unsigned grid_for(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)sm_count() * 8;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

}  // namespace sgs

using namespace sgs;

extern "C" int sgs_abi_version(void) { return SGS_ABI_VERSION; }
/* debug: per-column kernel timeline (8 x u64 per column), NULL disables */
extern "C" void sgs_debug_timeline(void* buf) {
  g_timeline = static_cast<unsigned long long*>(buf);
}
extern "C" void sgs_debug_timeline_col(int64_t col) { g_timeline_col = col; }
extern "C" const char* sgs_last_error(void) { return g_err; }
extern "C" uint64_t sgs_launch_count(void) { return g_launches.load(); }

extern "C" int sgs_device_sm_count(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
    set_error("cudaDeviceGetAttribute failed");
    return SGS_ECUDA;
  }
  return v;
}

extern "C" int sgs_status_init(sgs_status* st, void* stream) {
  SGS_REQUIRE(st, "status_init: null");
  status_init_kernel<<<1, 1, 0, as_stream(stream)>>>(st);
  return check_launch("status_init_kernel");
}

extern "C" int sgs_csr_spmv(int64_t n, const int32_t* row_ptr, const int32_t* col_idx,
                            const double* vals, const void* x, int x_dtype, const double* xdiv,
                            const double* alpha, double* y, const sgs_status* st, void* stream) {
  SGS_REQUIRE(n >= 1 && row_ptr && col_idx && vals && x && y, "spmv: bad args");
  // staging needs 16-byte aligned arrays (torch allocations are); else global loads
  const int stage = ((uintptr_t)col_idx & 15) == 0 && ((uintptr_t)vals & 15) == 0;
  cudaStream_t s = as_stream(stream);
  const unsigned blocks = (unsigned)((n + kSpRows - 1) / kSpRows);
  if (x_dtype == SGS_F32)
    return check_ex(launch_ex(csr_spmv_staged_kernel<float>, dim3(blocks), dim3(kSpThreads), 0, s,
                              1, n, row_ptr, col_idx, vals, static_cast<const float*>(x), xdiv,
                              alpha, y, st, debug_timeline_row(), stage),
                    "csr_spmv_staged_kernel");
  return check_ex(launch_ex(csr_spmv_staged_kernel<double>, dim3(blocks), dim3(kSpThreads), 0, s,
                            1, n, row_ptr, col_idx, vals, static_cast<const double*>(x), xdiv,
                            alpha, y, st, debug_timeline_row(), stage),
                  "csr_spmv_staged_kernel");
}

// Scratch of sgs_csr_spmv_srht for n local rows and k sample rows: tile
// vectors (doubles) and counters (u64, zeroed once by the caller).
extern "C" int64_t sgs_spmv_srht_tilevec_elems(int64_t n, int k) {
  return n < 1 || k < 1 ? 0 : (n + kSpTile - 1) / kSpTile * (int64_t)k;
}
extern "C" int64_t sgs_spmv_srht_counter_elems(int64_t n) {
  if (n < 1) return 0;
  const int64_t nt = (n + kSpTile - 1) / kSpTile;
  const int G = tile_group(n);
  return nt + (nt + G - 1) / G;
}

extern "C" int sgs_csr_spmv_srht(int64_t n, const int32_t* row_ptr, const int32_t* col_idx,
                                 const double* vals, const void* x, int x_dtype,
                                 const double* xdiv, const double* alpha, double* y, int64_t row0,
                                 int log2_block, const uint32_t* sign_bits,
                                 const int32_t* samples, int k, double* tilevec,
                                 unsigned long long* counters, double* partials,
                                 const sgs_status* st, void* stream) {
  SGS_REQUIRE(n >= 1 && row_ptr && col_idx && vals && x && y, "spmv_srht: bad args");
  SGS_REQUIRE(sign_bits && samples && tilevec && counters && partials && k >= 1 &&
                  k <= 8 * kSpThreads && log2_block >= 12 && log2_block <= 40 && row0 >= 0 &&
                  row0 % kSpTile == 0,
              "spmv_srht: bad sketch args (k <= %d, 4096-row tiles, tile-aligned row0)",
              8 * kSpThreads);
  const int stage = ((uintptr_t)col_idx & 15) == 0 && ((uintptr_t)vals & 15) == 0;
  cudaStream_t s = as_stream(stream);
  const unsigned blocks = (unsigned)((n + kSpRows - 1) / kSpRows);
  SpmvSrht sk;
  sk.row0 = row0;
  sk.log2_block = log2_block;
  sk.sign_bits = sign_bits;
  sk.samples = samples;
  sk.k = k;
  sk.G = tile_group(n);
  sk.tilevec = tilevec;
  sk.counters = counters;
  sk.partials = partials;
  const size_t a = (size_t)(kSpCap + 2) * 8 + (size_t)(kSpCap + 4) * 4;
  const size_t b = (size_t)kSpT3Buf * 8 + 128 * 4 + (size_t)k * 4;
  const size_t smem = a > b ? a : b;
#define SGS_SPSR_LAUNCH(TX, KQ)                                                              \
  do {                                                                                       \
    auto kern = csr_spmv_srht_kernel<TX, KQ>;                                                \
    if (smem > 48 * 1024)                                                                    \
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);    \
    return check_ex(launch_ex(kern, dim3(blocks), dim3(kSpThreads), smem, s, 1, n, row_ptr,  \
                              col_idx, vals, static_cast<const TX*>(x), xdiv, alpha, y, st,  \
                              debug_timeline_row(), stage, sk),                              \
                    "csr_spmv_srht_kernel");                                                 \
  } while (0)
  if (x_dtype == SGS_F32) {
    if (k <= 4 * kSpThreads) SGS_SPSR_LAUNCH(float, 4);
    SGS_SPSR_LAUNCH(float, 8);
  }
  if (k <= 4 * kSpThreads) SGS_SPSR_LAUNCH(double, 4);
  SGS_SPSR_LAUNCH(double, 8);
#undef SGS_SPSR_LAUNCH
}

extern "C" int64_t sgs_norm2_work_elems(int64_t n) { (void)n; return kNormBlocks; }

extern "C" int sgs_norm2(const void* x, int x_dtype, int64_t n, double* out, double* work,
                         void* stream) {
  SGS_REQUIRE(x && out && work && n >= 0, "norm2: bad args");
  cudaStream_t s = as_stream(stream);
  const int nb = kNormBlocks;
  if (x_dtype == SGS_F32)
    norm_partial_kernel<float><<<nb, 256, 0, s>>>(static_cast<const float*>(x), n, work);
  else
    norm_partial_kernel<double><<<nb, 256, 0, s>>>(static_cast<const double*>(x), n, work);
  int rc = check_launch("norm_partial_kernel");
  if (rc) return rc;
  norm_final_kernel<<<1, 256, 0, s>>>(work, nb, out);
  return check_launch("norm_final_kernel");
}

extern "C" int sgs_scale(const double* x, double num, const double* den, int divide, double* y,
                         int64_t n, void* stream) {
  SGS_REQUIRE(x && y && n >= 0 && (!divide || den), "scale: bad args");
  if (n == 0) return SGS_OK;
  scale_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(x, num, den, divide, y, n);
  return check_launch("scale_kernel");
}

extern "C" int sgs_rsub(const double* b, double* y, int64_t n, void* stream) {
  SGS_REQUIRE(b && y && n >= 0, "rsub: bad args");
  if (n == 0) return SGS_OK;
  rsub_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(b, y, n);
  return check_launch("rsub_kernel");
}

extern "C" int sgs_cast_div(const void* src, int src_dtype, void* dst, int dst_dtype,
                            const double* den, int64_t n, void* stream) {
  SGS_REQUIRE(src && dst && n >= 0, "cast_div: bad args");
  if (n == 0) return SGS_OK;
  cudaStream_t s = as_stream(stream);
  const unsigned g = grid_for(n);
  if (src_dtype == SGS_F64 && dst_dtype == SGS_F64)
    cast_div_kernel<double, double><<<g, 256, 0, s>>>(static_cast<const double*>(src), den,
                                                       static_cast<double*>(dst), n);
  else if (src_dtype == SGS_F64 && dst_dtype == SGS_F32)
    cast_div_kernel<double, float><<<g, 256, 0, s>>>(static_cast<const double*>(src), den,
                                                      static_cast<float*>(dst), n);
  else if (src_dtype == SGS_F32 && dst_dtype == SGS_F64)
    cast_div_kernel<float, double><<<g, 256, 0, s>>>(static_cast<const float*>(src), den,
                                                      static_cast<double*>(dst), n);
  else
    cast_div_kernel<float, float><<<g, 256, 0, s>>>(static_cast<const float*>(src), den,
                                                     static_cast<float*>(dst), n);
  return check_launch("cast_div_kernel");
}

extern "C" int sgs_cos_init(double* v, int64_t n, void* stream) {
  return sgs_cos_init_at(v, n, 0, stream);
}

extern "C" int sgs_cos_init_at(double* v, int64_t n, int64_t first, void* stream) {
  SGS_REQUIRE(v && n >= 0 && first >= 0, "cos_init: bad args");
  if (n == 0) return SGS_OK;
  cos_init_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(v, n, first);
  return check_launch("cos_init_kernel");
}

extern "C" int sgs_power_step(const double* w, const double* nrm, double* v, double* sigma,
                              int64_t n, void* stream) {
  SGS_REQUIRE(w && nrm && v && sigma && n >= 1, "power_step: bad args");
  cudaStream_t s = as_stream(stream);
  power_commit_kernel<<<1, 1, 0, s>>>(nrm, sigma);
  int rc = check_launch("power_commit_kernel");
  if (rc) return rc;
  power_step_kernel<<<grid_for(n), 256, 0, s>>>(w, nrm, v, sigma, n);
  return check_launch("power_step_kernel");
}

extern "C" int sgs_arnoldi_head(void* Q, int q_dtype, int64_t ldq, int64_t n, int col,
                                const double* R, int64_t ldr, int* norm_flag, int gi, double* cs,
                                double* sn, double* g, double* T, int64_t ldt, double* hist,
                                double tol, sgs_status* st, void* stream) {
  SGS_REQUIRE(R && st && n >= 1 && (col < 0 || (Q && norm_flag && ldq >= n && col < ldr)),
              "arnoldi_head: bad args");
  SGS_REQUIRE(gi < 0 || (cs && sn && g && T && hist && ldr >= gi + 2 && ldt >= gi + 2 &&
                         gi + 2 <= kGivMax),
              "arnoldi_head: bad Givens args");
  const size_t smem = gi >= 0 ? (size_t)(3 * gi + 2) * sizeof(double) : 0;
  const unsigned nb = (col >= 0 ? (unsigned)((n + 256 * kHeadPer - 1) / (256 * kHeadPer)) : 0) +
                      (gi >= 0 ? 1 : 0);
  if (nb == 0) return SGS_OK;
  cudaStream_t s = as_stream(stream);
  if (q_dtype == SGS_F32) {
    auto kern = arnoldi_head_kernel<float>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return check_ex(launch_ex(kern, dim3(nb), dim3(256), smem, s, 1, static_cast<float*>(Q), ldq, n,
                              col, norm_flag, gi, R, ldr, cs, sn, g, T, ldt, hist, tol, st,
                              debug_timeline()),
                    "arnoldi_head_kernel");
  }
  auto kern = arnoldi_head_kernel<double>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return check_ex(launch_ex(kern, dim3(nb), dim3(256), smem, s, 1, static_cast<double*>(Q), ldq, n,
                            col, norm_flag, gi, R, ldr, cs, sn, g, T, ldt, hist, tol, st,
                            debug_timeline()),
                  "arnoldi_head_kernel");
}

extern "C" int sgs_givens_step(const double* R, int64_t ldr, int i, double* cs, double* sn,
                               double* g, double* T, int64_t ldt, double* hist, double tol,
                               sgs_status* st, void* stream) {
  SGS_REQUIRE(R && cs && sn && g && T && hist && st && i >= 0 && ldr >= i + 2 && ldt >= i + 2,
              "givens: bad args");
  SGS_REQUIRE(i + 2 <= kGivMax, "givens: restart length %d too large", i + 2);
  const size_t smem = (size_t)(3 * i + 2) * sizeof(double);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(givens_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return check_ex(launch_ex(givens_step_kernel, dim3(1), dim3(256), smem, as_stream(stream), 1, R,
                            ldr, i, cs, sn, g, T, ldt, hist, tol, st, debug_timeline()),
                  "givens_step_kernel");
}
