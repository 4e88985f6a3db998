// ILU(0) right preconditioner on the device (reference krylov.py:86-151).
//
// Both the factorization and the two triangular sweeps are dependency-driven
// ("sync-free") row kernels: one thread per row, row blocks handed out in
// order by an atomic ticket (so every row a thread waits for belongs to a
// block that is already resident - no deadlock, no level analysis), and a
// per-row readiness flag published with st.release / polled with ld.acquire.
// The critical path is the matrix's dependency depth (3*128-2 rows for the
// 128^3 7-point stencil), each hop one L2 round trip.
#include "sgs_common.cuh"

namespace sgs {
namespace {

constexpr int kIluThreads = 128;

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_ready(const uint32_t* flag, uint32_t want) {
  if (ld_acquire(flag) == want) return;
  while (ld_acquire(flag) != want) __nanosleep(20);
}

// Claims the block's ticket (rows [t*blockDim, (t+1)*blockDim) in sweep
// order) and the launch epoch.  Every block takes a ticket, even one that
// returns early, so the last-block bookkeeping stays exact.
struct Claim {
  int64_t first;
  uint32_t want;
};
__device__ __forceinline__ Claim claim_rows(sgs_ilu_ctl* ctl) {
  __shared__ int64_t s_first;
  __shared__ uint32_t s_want;
  if (threadIdx.x == 0) {
    const unsigned long long t = atomicAdd(reinterpret_cast<unsigned long long*>(&ctl->ticket), 1ull);
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

// Row i of the IKJ elimination (krylov.py:126-145), in the reference's
// storage order and rounding: lik = a_ik / u_kk, a_ij -= lik * u_kj for the
// entries of row i after k that row k also holds.
__global__ void __launch_bounds__(kIluThreads)
ilu_factor_kernel(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                  double* F, const int32_t* __restrict__ diag_pos, uint32_t* flags,
                  sgs_ilu_ctl* ctl, unsigned long long* aux, double pivot_tol) {
  const Claim c = claim_rows(ctl);
  const bool structural = *reinterpret_cast<volatile unsigned long long*>(aux) != (unsigned long long)n;
  const int64_t i = c.first + threadIdx.x;
  if (!structural && i < n) {
    const int lo = rp[i], hi = rp[i + 1];
    if (i >= 1) {
      for (int p = lo; p < hi; ++p) {
        const int k = ci[p];
        if (k >= i) break;
        wait_ready(flags + k, c.want);
        const double pivot = __ldcg(F + diag_pos[k]);
        if (fabs(pivot) < pivot_tol) atomicMin(aux + 1, 2ull * (unsigned long long)i);
        const double lik = __ddiv_rn(F[p], pivot);
        F[p] = lik;
        const int klo = rp[k], khi = rp[k + 1];
        for (int q = p + 1; q < hi; ++q) {
          const int j = ci[q];
          int pos = -1;
          for (int t = klo; t < khi; ++t)
            if (ci[t] == j) pos = t;
          if (pos >= 0) F[q] = __dsub_rn(F[q], __dmul_rn(lik, __ldcg(F + pos)));
        }
      }
      if (fabs(F[diag_pos[i]]) < pivot_tol) atomicMin(aux + 1, 2ull * (unsigned long long)i + 1ull);
    }
    st_release(flags + i, c.want);
  }
  retire_block(ctl);
}

// One triangular sweep.  kLower: tmp_i = x_i - sum_{j<i} F_ij tmp_j (unit
// diagonal); else out_i = (tmp_i - sum_{j>i} F_ij out_j) / F_ii, rows in
// descending order.
template <typename TX, bool kLower>
__global__ void __launch_bounds__(kIluThreads)
ilu_sweep_kernel(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                 const double* __restrict__ F, const int32_t* __restrict__ diag_pos,
                 const TX* __restrict__ x, const double* __restrict__ xdiv, double* out,
                 uint32_t* flags, sgs_ilu_ctl* ctl, const sgs_status* st) {
  const Claim c = claim_rows(ctl);
  const int64_t r = c.first + threadIdx.x;
  if (!status_stopped(st) && r < n) {
    const int64_t i = kLower ? r : n - 1 - r;
    double acc;
    if (xdiv != nullptr) {
      const double v = (double)__ldg(x + i) / __ldg(xdiv);
      if constexpr (sizeof(TX) == 4) acc = (double)__double2float_rn(v);
      else acc = v;
    } else {
      acc = (double)__ldg(x + i);
    }
    const int lo = __ldg(rp + i), hi = __ldg(rp + i + 1);
    for (int p = lo; p < hi; ++p) {
      const int j = __ldg(ci + p);
      if (kLower ? (j < i) : (j > i)) {
        wait_ready(flags + j, c.want);
        acc = fma(-__ldg(F + p), __ldcg(out + j), acc);
      }
    }
    if (!kLower) acc = acc / __ldg(F + __ldg(diag_pos + i));
    __stcg(out + i, acc);
    st_release(flags + i, c.want);
  }
  retire_block(ctl);
}

inline unsigned blocks_for(int64_t n) { return (unsigned)((n + kIluThreads - 1) / kIluThreads); }

}  // namespace
}  // namespace sgs

using namespace sgs;

extern "C" int sgs_ilu0_factor(int64_t n, const int32_t* rp, const int32_t* ci, const double* vals,
                               double* F, int32_t* diag_pos, uint32_t* flags, sgs_ilu_ctl* ctl,
                               uint64_t* aux, double pivot_tol, void* stream) {
  SGS_REQUIRE(n >= 0 && (n == 0 || (rp && ci && vals && F && diag_pos && flags && ctl && aux)),
              "ilu0_factor: bad args");
  if (n == 0) return SGS_OK;
  cudaStream_t s = as_stream(stream);
  unsigned long long* a = reinterpret_cast<unsigned long long*>(aux);
  ilu_aux_init_kernel<<<1, 1, 0, s>>>(n, a);
  int rc = check_launch("ilu_aux_init_kernel");
  if (rc) return rc;
  ilu_diag_kernel<<<blocks_for(n), kIluThreads, 0, s>>>(n, rp, ci, vals, F, diag_pos, a);
  rc = check_launch("ilu_diag_kernel");
  if (rc) return rc;
  ilu_factor_kernel<<<blocks_for(n), kIluThreads, 0, s>>>(
      n, rp, ci, F, diag_pos, flags, ctl, a, pivot_tol);
  return check_launch("ilu_factor_kernel");
}

extern "C" int sgs_ilu0_solve(int64_t n, const int32_t* rp, const int32_t* ci, const double* F,
                              const int32_t* diag_pos, const void* x, int x_dtype,
                              const double* xdiv, double* tmp, double* out, uint32_t* flags,
                              sgs_ilu_ctl* ctl, const sgs_status* st, void* stream) {
  SGS_REQUIRE(n >= 0 && (n == 0 || (rp && ci && F && diag_pos && x && tmp && out && flags && ctl)),
              "ilu0_solve: bad args");
  SGS_REQUIRE(x_dtype == SGS_F32 || x_dtype == SGS_F64, "ilu0_solve: bad dtype");
  SGS_REQUIRE(tmp != out && (const void*)tmp != x, "ilu0_solve: tmp must not alias x or out");
  if (n == 0) return SGS_OK;
  cudaStream_t s = as_stream(stream);
  const unsigned nb = blocks_for(n);
  if (x_dtype == SGS_F32)
    ilu_sweep_kernel<float, true><<<nb, kIluThreads, 0, s>>>(
        n, rp, ci, F, diag_pos, static_cast<const float*>(x), xdiv, tmp, flags, ctl, st);
  else
    ilu_sweep_kernel<double, true><<<nb, kIluThreads, 0, s>>>(
        n, rp, ci, F, diag_pos, static_cast<const double*>(x), xdiv, tmp, flags, ctl, st);
  int rc = check_launch("ilu_sweep_kernel<lower>");
  if (rc) return rc;
  ilu_sweep_kernel<double, false><<<nb, kIluThreads, 0, s>>>(n, rp, ci, F, diag_pos, tmp, nullptr,
                                                             out, flags, ctl, st);
  return check_launch("ilu_sweep_kernel<upper>");
}
