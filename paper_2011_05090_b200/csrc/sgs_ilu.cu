// ILU(0) right preconditioner on the device (reference krylov.py:86-151).
//
// Analysis: every row gets its dependency level in the lower (j < i) and the
// upper (j > i) triangle, and the rows are counting-sorted by level into two
// permutations.  The factorization and the triangular sweeps are then
// dependency-driven ("sync-free") row kernels that hand rows out in LEVEL
// order through an atomic ticket: every row a thread waits for has a lower
// level, hence an earlier ticket, hence a resident (or finished) thread - no
// deadlock - and the resident window follows the wavefront instead of the
// row order (in row order the 128^3 stencil's wavefront spans ~130 z-planes
// while only ~7 fit on the GPU, which serialises the sweep ~20x).
//
// Readiness: the sweeps poll the VALUE itself.  Outputs hold a signalling-NaN
// sentinel until written (no arithmetic result is a signalling NaN, and the
// one pass-through value is canonicalised), so one 8-byte relaxed load both
// waits and reads - no flag array and no release fence on the critical path.
// The forward sweep re-arms `out` and the backward sweep re-arms `tmp` behind
// itself, so consecutive solves need no fill launches.  The factorization
// publishes whole rows and keeps a per-row epoch flag (release / acquire).
#include "sgs_common.cuh"

#include <cstdlib>

namespace sgs {
namespace {

constexpr int kIluThreads = 128;
constexpr int kRowChunk = 8;
constexpr unsigned long long kPending = 0x7FF400005EED0001ull;  // signalling NaN

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed_i(const int32_t* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_b64(const double* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_b64(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(__double_as_longlong(v))
               : "memory");
}
__device__ __forceinline__ void st_relaxed_i(int32_t* p, int v) {
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ double pending_value() { return __longlong_as_double((long long)kPending); }
__device__ __forceinline__ double publishable(double v) {
  return (unsigned long long)__double_as_longlong(v) == kPending ? __longlong_as_double(0x7FF8000000000000ll)
                                                                  : v;
}

// Claims the block's ticket: positions [t*blockDim, (t+1)*blockDim) of the
// launch's row order.  Every block takes one, even one that returns early,
// so the last-block bookkeeping stays exact.
struct Claim {
  int64_t first;
  uint32_t want;
};
__device__ __forceinline__ Claim claim_rows(sgs_ilu_ctl* ctl) {
  __shared__ int64_t s_first;
  __shared__ uint32_t s_want;
  if (threadIdx.x == 0) {
    const unsigned long long t =
        atomicAdd(reinterpret_cast<unsigned long long*>(&ctl->ticket), 1ull);
    s_first = (int64_t)t * blockDim.x;
    s_want = *reinterpret_cast<volatile uint32_t*>(&ctl->epoch) + 1u;
  }
  __syncthreads();
  return {s_first, s_want};
}

// The last block of a launch resets the ticket and advances the epoch.
__device__ __forceinline__ void retire_block(sgs_ilu_ctl* ctl) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t prev = atomicAdd(&ctl->done, 1u);
    if (prev == gridDim.x - 1) {
      ctl->ticket = 0;
      ctl->done = 0;
      __threadfence();
      atomicAdd(&ctl->epoch, 1u);
    }
  }
}

__global__ void fill_i32_kernel(int32_t* p, int64_t n, int v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}
__global__ void fill_pending_kernel(double* p, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = pending_value();
}

// ---- analysis -----------------------------------------------------------------
// lev[i] = 1 + max lev[j] over the row's dependencies (0 without any), in row
// order (ascending for the lower triangle, descending for the upper), warp-
// cooperative: dependencies in earlier warps are polled (lev holds -1 until
// written), dependencies inside the warp are resolved by a shuffle chain.
template <bool kLower>
__global__ void __launch_bounds__(kIluThreads)
ilu_level_kernel(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                 int32_t* lev, sgs_ilu_ctl* ctl) {
  const Claim c = claim_rows(ctl);
  const int lane = threadIdx.x & 31;
  const int64_t wbase = c.first + (int64_t)(threadIdx.x >> 5) * 32;
  const int64_t r = wbase + lane;
  int my = 0;
  uint32_t deps = 0;
  int64_t i = -1;
  if (r < n) {
    i = kLower ? r : n - 1 - r;
    const int lo = __ldg(rp + i), hi = __ldg(rp + i + 1);
    for (int base = lo; base < hi; base += kRowChunk) {
      int64_t cj[kRowChunk];
#pragma unroll
      for (int u = 0; u < kRowChunk; ++u) cj[u] = base + u < hi ? (int64_t)__ldg(ci + base + u) : -1;
      uint32_t ext = 0;
#pragma unroll
      for (int u = 0; u < kRowChunk; ++u) {
        const int64_t j = cj[u];
        if (j >= 0 && (kLower ? (j < i) : (j > i))) {
          const int64_t rj = kLower ? j : n - 1 - j;
          if (rj >= wbase) deps |= 1u << (rj - wbase);
          else ext |= 1u << u;
        }
      }
      while (ext) {
#pragma unroll
        for (int u = 0; u < kRowChunk; ++u)
          if ((ext >> u) & 1u) {
            const int l = ld_relaxed_i(lev + cj[u]);
            if (l >= 0) {
              my = max(my, l + 1);
              ext &= ~(1u << u);
            }
          }
      }
    }
  }
  __syncwarp();
  uint32_t need = __reduce_or_sync(0xffffffffu, deps);
  while (need) {
    const int t = __ffs(need) - 1;
    need &= need - 1;
    const int lt = __shfl_sync(0xffffffffu, my, t);
    if ((deps >> t) & 1u) my = max(my, lt + 1);
  }
  if (r < n) st_relaxed_i(lev + i, my);
  retire_block(ctl);
}

__global__ void level_hist_kernel(const int32_t* __restrict__ lev, int64_t n, int32_t* hist,
                                  int32_t* maxlev) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int l = lev[i];
    atomicAdd(hist + l, 1);
    atomicMax(maxlev, l);
  }
}

// Exclusive scan of hist[0..maxlev] in place (one block; levels are few).
__global__ void __launch_bounds__(1024) level_scan_kernel(int32_t* hist, const int32_t* maxlev) {
  __shared__ int32_t warp_tot[32];
  __shared__ int32_t carry;
  const int64_t L = (int64_t)*maxlev + 1;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t base = 0; base < L; base += 1024) {
    const int64_t idx = base + threadIdx.x;
    const int v = idx < L ? hist[idx] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    if (w == 0) {
      int t = warp_tot[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      warp_tot[lane] = t;  // inclusive
    }
    __syncthreads();
    const int before = carry + (w ? warp_tot[w - 1] : 0) + incl - v;
    if (idx < L) hist[idx] = before;
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_tot[31];
    __syncthreads();
  }
}

__global__ void level_scatter_kernel(const int32_t* __restrict__ lev, int64_t n, int32_t* off,
                                     int32_t* perm) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    perm[atomicAdd(off + lev[i], 1)] = (int32_t)i;
}

// ---- factorization ----------------------------------------------------------------
__global__ void ilu_aux_init_kernel(int64_t n, unsigned long long* aux) {
  aux[0] = (unsigned long long)n;
  aux[1] = ~0ull;
}

// F = vals; diag_pos[i] = position of column i in row i (the last one, as
// the reference's {col: pos} dict keeps); aux[0] = min row without one.
__global__ void ilu_diag_kernel(int64_t n, const int32_t* __restrict__ rp,
                                const int32_t* __restrict__ ci, const double* __restrict__ vals,
                                double* __restrict__ F, int32_t* __restrict__ diag_pos,
                                unsigned long long* aux) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int d = -1;
  for (int p = rp[i]; p < rp[i + 1]; ++p) {
    F[p] = vals[p];
    if (ci[p] == i) d = p;
  }
  diag_pos[i] = d;
  if (d < 0) atomicMin(aux, (unsigned long long)i);
}

__device__ __forceinline__ void wait_flag(const uint32_t* flag, uint32_t want) {
  while (ld_relaxed(flag) != want) {
  }
  (void)ld_acquire(flag);
}

// Generic row of the IKJ elimination (any row length), straight from memory,
// starting at entry p0 (entries before it already eliminated).
__device__ void factor_row_generic_from(int64_t i, int p0, int lo, int hi, const int32_t* __restrict__ rp,
                                   const int32_t* __restrict__ ci, double* F,
                                   const int32_t* __restrict__ diag_pos, const uint32_t* flags,
                                   uint32_t want, unsigned long long* aux, double pivot_tol) {
  (void)lo;
  for (int p = p0; p < hi; ++p) {
    const int k = ci[p];
    if (k >= i) break;
    wait_flag(flags + k, want);
    const double pivot = __ldcg(F + diag_pos[k]);
    if (fabs(pivot) < pivot_tol) atomicMin(aux + 1, 2ull * (unsigned long long)i);
    const double lik = __ddiv_rn(F[p], pivot);
    F[p] = lik;
    const int klo = rp[k], khi = rp[k + 1];
    for (int q = p + 1; q < hi; ++q) {
      const int j = ci[q];
      int at = -1;
      for (int t = klo; t < khi; ++t)
        if (ci[t] == j) at = t;
      if (at >= 0) F[q] = __dsub_rn(F[q], __dmul_rn(lik, __ldcg(F + at)));
    }
  }
  if (fabs(F[diag_pos[i]]) < pivot_tol) atomicMin(aux + 1, 2ull * (unsigned long long)i + 1ull);
}

constexpr int kFacMax = 12;  // rows (and pivot rows) up to this length run from registers

// Row i of the IKJ elimination (krylov.py:126-145), in the reference's
// storage order and rounding: lik = a_ik / u_kk, a_ij -= lik * u_kj for the
// entries of row i after k that row k also holds.  Rows in lower-level
// order.  Short rows keep the row in registers and load each pivot row in
// one batch (its column indices before the wait, its values after), so a
// row costs a few memory latencies instead of one per scanned entry.
__global__ void __launch_bounds__(kIluThreads)
ilu_factor_kernel(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                  double* F, const int32_t* __restrict__ diag_pos,
                  const int32_t* __restrict__ perm, uint32_t* flags, sgs_ilu_ctl* ctl,
                  unsigned long long* aux, double pivot_tol) {
  const Claim c = claim_rows(ctl);
  const bool structural =
      *reinterpret_cast<volatile unsigned long long*>(aux) != (unsigned long long)n;
  const int64_t pos = c.first + threadIdx.x;
  if (!structural && pos < n) {
    const int64_t i = __ldg(perm + pos);
    const int lo = __ldg(rp + i), hi = __ldg(rp + i + 1);
    const int len = hi - lo;
    if (i >= 1 && len > kFacMax) {
      factor_row_generic_from(i, lo, lo, hi, rp, ci, F, diag_pos, flags, c.want, aux, pivot_tol);
    } else if (i >= 1) {
      int oc[kFacMax];
      double of[kFacMax];
#pragma unroll
      for (int u = 0; u < kFacMax; ++u) {
        oc[u] = u < len ? __ldg(ci + lo + u) : INT32_MAX;
        of[u] = u < len ? F[lo + u] : 0.0;
      }
      // pivots: the leading entries with column < i (the reference breaks at
      // the first column >= i, krylov.py:129-130)
      int npiv = 0;
      bool open = true;
#pragma unroll
      for (int u = 0; u < kFacMax; ++u) {
        open = open && oc[u] < i;
        npiv += open ? 1 : 0;
      }
      bool generic = false;
#pragma unroll
      for (int u = 0; u < kFacMax; ++u) {
        if (u >= npiv || generic) continue;
        const int k = oc[u];
        const int klo = __ldg(rp + k), khi = __ldg(rp + k + 1);
        if (khi - klo > kFacMax) {
          generic = true;  // finish this row from memory (rare: long pivot row)
          continue;
        }
        int kc[kFacMax];
#pragma unroll
        for (int t = 0; t < kFacMax; ++t) kc[t] = t < khi - klo ? __ldg(ci + klo + t) : -1;
        wait_flag(flags + k, c.want);
        double kf[kFacMax];
#pragma unroll
        for (int t = 0; t < kFacMax; ++t) kf[t] = t < khi - klo ? __ldcg(F + klo + t) : 0.0;
        double pivot = 0.0;
#pragma unroll
        for (int t = 0; t < kFacMax; ++t)
          if (kc[t] == k) pivot = kf[t];  // last occurrence, as diag_pos
        if (fabs(pivot) < pivot_tol) atomicMin(aux + 1, 2ull * (unsigned long long)i);
        const double lik = __ddiv_rn(of[u], pivot);
        of[u] = lik;
#pragma unroll
        for (int q = 0; q < kFacMax; ++q) {
          if (q <= u || q >= len) continue;
          double kv = 0.0;
          bool hit = false;
#pragma unroll
          for (int t = 0; t < kFacMax; ++t)
            if (kc[t] == oc[q]) {
              kv = kf[t];
              hit = true;
            }
          if (hit) of[q] = __dsub_rn(of[q], __dmul_rn(lik, kv));
        }
      }
#pragma unroll
      for (int u = 0; u < kFacMax; ++u)
        if (u < len) F[lo + u] = of[u];
      if (generic) {
        // redo from the first unprocessed pivot with the generic loop: the
        // registers already hold pivots [0, done) applied and written back
        int done = 0;
#pragma unroll
        for (int u = 0; u < kFacMax; ++u) {
          if (u < npiv) {
            const int k = oc[u];
            if (__ldg(rp + k + 1) - __ldg(rp + k) > kFacMax) break;
            ++done;
          }
        }
        factor_row_generic_from(i, lo + done, lo, hi, rp, ci, F, diag_pos, flags, c.want, aux,
                                pivot_tol);
      } else {
        double dv = 0.0;
#pragma unroll
        for (int u = 0; u < kFacMax; ++u)
          if (u < len && oc[u] == i) dv = of[u];
        if (fabs(dv) < pivot_tol) atomicMin(aux + 1, 2ull * (unsigned long long)i + 1ull);
      }
    }
    st_release(flags + i, c.want);
  }
  retire_block(ctl);
}

// ---- triangular sweeps ----------------------------------------------------------
// One row per thread in level order.
//   kLower: tmp_i = x_i - sum_{j<i} F_ij tmp_j   (unit diagonal); re-arms out_i
//   upper : out_i = (tmp_i - sum_{j>i} F_ij out_j) / F_ii;   re-arms tmp_i
// `dst` is the array written (and polled), `rearm` the one re-armed.
template <typename TX, bool kLower>
__global__ void __launch_bounds__(kIluThreads)
ilu_sweep_kernel(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                 const double* __restrict__ F, const int32_t* __restrict__ perm,
                 const TX* x, const double* __restrict__ xdiv, double* dst, double* rearm,
                 sgs_ilu_ctl* ctl, const sgs_status* st, unsigned sleep_ns) {
  const Claim c = claim_rows(ctl);
  const int64_t pos = c.first + threadIdx.x;
  if (!status_stopped(st) && pos < n) {
    const int64_t i = __ldg(perm + pos);
    double acc, dinv = 1.0;
    if (kLower && xdiv != nullptr) {
      const double v = (double)__ldg(x + i) / __ldg(xdiv);
      if constexpr (sizeof(TX) == 4) acc = (double)__double2float_rn(v);
      else acc = v;
    } else {
      acc = (double)x[i];
    }
    const int lo = __ldg(rp + i), hi = __ldg(rp + i + 1);
    for (int base = lo; base < hi; base += kRowChunk) {
      int64_t cj[kRowChunk];
      double cf[kRowChunk], v[kRowChunk];
#pragma unroll
      for (int u = 0; u < kRowChunk; ++u) {
        const int p = base + u;
        cj[u] = p < hi ? (int64_t)__ldg(ci + p) : -1;
        cf[u] = p < hi ? __ldg(F + p) : 0.0;
      }
      uint32_t ext = 0;
#pragma unroll
      for (int u = 0; u < kRowChunk; ++u) {
        const int64_t j = cj[u];
        if (j < 0) continue;
        if (kLower ? (j < i) : (j > i)) ext |= 1u << u;
        else if (!kLower && j == i) dinv = 1.0 / cf[u];
      }
      uint32_t pend = ext;
      while (true) {
#pragma unroll
        for (int u = 0; u < kRowChunk; ++u)
          if ((pend >> u) & 1u) {
            const unsigned long long b = ld_relaxed_b64(dst + cj[u]);
            if (b != kPending) {
              v[u] = __longlong_as_double((long long)b);
              pend &= ~(1u << u);
            }
          }
        if (!pend) break;
        if (sleep_ns) __nanosleep(sleep_ns);
      }
#pragma unroll
      for (int u = 0; u < kRowChunk; ++u)
        if ((ext >> u) & 1u) acc = fma(-cf[u], v[u], acc);
    }
    if (!kLower) acc *= dinv;
    rearm[i] = pending_value();
    st_relaxed_b64(dst + i, publishable(acc));
  }
  retire_block(ctl);
}

inline unsigned sweep_sleep_ns() {
  static const unsigned v = [] {
    const char* e = getenv("SGS_ILU_SLEEP_NS");
    return e ? (unsigned)atoi(e) : 0u;
  }();
  return v;
}

inline unsigned blocks_for(int64_t n) { return (unsigned)((n + kIluThreads - 1) / kIluThreads); }
inline unsigned fill_blocks(int64_t n) {
  return (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
}

}  // namespace
}  // namespace sgs

using namespace sgs;

extern "C" int64_t sgs_ilu0_analysis_work_elems(int64_t n) { return 3 * n + 8; }

extern "C" int sgs_ilu0_analyse(int64_t n, const int32_t* rp, const int32_t* ci,
                                int32_t* perm_lower, int32_t* perm_upper, int32_t* work,
                                sgs_ilu_ctl* ctl, void* stream) {
  SGS_REQUIRE(n >= 0 && n < (int64_t)INT32_MAX &&
                  (n == 0 || (rp && ci && perm_lower && perm_upper && work && ctl)),
              "ilu0_analyse: bad args");
  if (n == 0) return SGS_OK;
  cudaStream_t s = as_stream(stream);
  int32_t* lev = work;           // n
  int32_t* hist = work + n;      // n + 1
  int32_t* maxlev = work + 2 * n + 1;
  for (int tri = 0; tri < 2; ++tri) {
    int32_t* perm = tri == 0 ? perm_lower : perm_upper;
    fill_i32_kernel<<<fill_blocks(n), 256, 0, s>>>(lev, n, -1);
    fill_i32_kernel<<<fill_blocks(n + 2), 256, 0, s>>>(hist, n + 2, 0);
    int rc = check_launch("fill_i32_kernel");
    if (rc) return rc;
    if (tri == 0)
      ilu_level_kernel<true><<<blocks_for(n), kIluThreads, 0, s>>>(n, rp, ci, lev, ctl);
    else
      ilu_level_kernel<false><<<blocks_for(n), kIluThreads, 0, s>>>(n, rp, ci, lev, ctl);
    if ((rc = check_launch("ilu_level_kernel"))) return rc;
    level_hist_kernel<<<fill_blocks(n), 256, 0, s>>>(lev, n, hist, maxlev);
    if ((rc = check_launch("level_hist_kernel"))) return rc;
    level_scan_kernel<<<1, 1024, 0, s>>>(hist, maxlev);
    if ((rc = check_launch("level_scan_kernel"))) return rc;
    level_scatter_kernel<<<fill_blocks(n), 256, 0, s>>>(lev, n, hist, perm);
    if ((rc = check_launch("level_scatter_kernel"))) return rc;
  }
  return SGS_OK;
}

extern "C" int sgs_ilu0_factor(int64_t n, const int32_t* rp, const int32_t* ci, const double* vals,
                               double* F, int32_t* diag_pos, const int32_t* perm_lower,
                               uint32_t* flags, sgs_ilu_ctl* ctl, uint64_t* aux, double pivot_tol,
                               void* stream) {
  SGS_REQUIRE(n >= 0 && (n == 0 || (rp && ci && vals && F && diag_pos && perm_lower && flags &&
                                    ctl && aux)),
              "ilu0_factor: bad args");
  if (n == 0) return SGS_OK;
  cudaStream_t s = as_stream(stream);
  unsigned long long* a = reinterpret_cast<unsigned long long*>(aux);
  ilu_aux_init_kernel<<<1, 1, 0, s>>>(n, a);
  int rc = check_launch("ilu_aux_init_kernel");
  if (rc) return rc;
  ilu_diag_kernel<<<blocks_for(n), kIluThreads, 0, s>>>(n, rp, ci, vals, F, diag_pos, a);
  if ((rc = check_launch("ilu_diag_kernel"))) return rc;
  ilu_factor_kernel<<<blocks_for(n), kIluThreads, 0, s>>>(n, rp, ci, F, diag_pos, perm_lower,
                                                          flags, ctl, a, pivot_tol);
  return check_launch("ilu_factor_kernel");
}

extern "C" int sgs_ilu0_pending_fill(double* v, int64_t n, void* stream) {
  SGS_REQUIRE(n >= 0 && (n == 0 || v), "ilu0_pending_fill: bad args");
  if (n == 0) return SGS_OK;
  fill_pending_kernel<<<fill_blocks(n), 256, 0, as_stream(stream)>>>(v, n);
  return check_launch("fill_pending_kernel");
}

extern "C" int sgs_ilu0_solve(int64_t n, const int32_t* rp, const int32_t* ci, const double* F,
                              const int32_t* perm_lower, const int32_t* perm_upper, const void* x,
                              int x_dtype, const double* xdiv, double* tmp, double* out,
                              sgs_ilu_ctl* ctl, const sgs_status* st, void* stream) {
  SGS_REQUIRE(n >= 0 && (n == 0 || (rp && ci && F && perm_lower && perm_upper && x && tmp && out &&
                                    ctl)),
              "ilu0_solve: bad args");
  SGS_REQUIRE(x_dtype == SGS_F32 || x_dtype == SGS_F64, "ilu0_solve: bad dtype");
  SGS_REQUIRE(tmp != out && (const void*)tmp != x && (const void*)out != x,
              "ilu0_solve: x, tmp and out must be distinct");
  if (n == 0) return SGS_OK;
  cudaStream_t s = as_stream(stream);
  const unsigned nb = blocks_for(n);
  if (x_dtype == SGS_F32)
    ilu_sweep_kernel<float, true><<<nb, kIluThreads, 0, s>>>(
        n, rp, ci, F, perm_lower, static_cast<const float*>(x), xdiv, tmp, out, ctl, st, sweep_sleep_ns());
  else
    ilu_sweep_kernel<double, true><<<nb, kIluThreads, 0, s>>>(
        n, rp, ci, F, perm_lower, static_cast<const double*>(x), xdiv, tmp, out, ctl, st, sweep_sleep_ns());
  int rc = check_launch("ilu_sweep_kernel<lower>");
  if (rc) return rc;
  ilu_sweep_kernel<double, false><<<nb, kIluThreads, 0, s>>>(n, rp, ci, F, perm_upper, tmp,
                                                             nullptr, out, tmp, ctl, st,
                                                             sweep_sleep_ns());
  return check_launch("ilu_sweep_kernel<upper>");
}
