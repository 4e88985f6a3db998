// Grid-wide sketched least-squares step (sm_100a).
//
// Same contract as the cluster kernel in sgs_rgs.cu (sgs_ls_step), but spread
// over one CTA per SM so the k-dimensional state (T = unnormalised orthogonal
// factor of S, R_S^{-1}) is read with the L2 bandwidth of the whole chip.
// The k rows are split over G CTAs (~10 rows each at k = 1500); every cross-CTA
// reduction is a reduce-scatter (each CTA sums a slice of entries over the G
// per-CTA partials, ascending CTA order) followed by an all-gather, separated
// by software grid barriers.  A fused finalize(i) + solve(i+1) launch needs
// three barriers:
//   B1  per-CTA partials of ||s'||^2, ||p_i||^2, T^T s', T^T p_{i+1}
//   B2  reduced entries (reduce-scatter done)
//   B3  per-CTA partials of ||t||^2 and t^T p_{i+1}
// Each entry is reduced by the same code wherever it sits, so streaming push
// and the batched factorisation agree bit for bit.  All CTAs must be
// co-resident: G <= #SMs, one 512-thread CTA per SM, and with programmatic
// dependent launch the successor grid is admitted only after every CTA of
// this grid has started.

#include "sgs_common.cuh"

namespace sgs {

constexpr int kLgThreads = 512;
constexpr int kLgMinRows = 8;
constexpr int kLgMaxG = 160;
constexpr int kLgSub = 64;  // threads per reduced entry in the reduce-scatter

// ---- software grid barrier ---------------------------------------------------
// bar[0] = arrival count, bar[1] = generation.  Every CTA reads the generation
// at kernel start (nobody can bump it before all CTAs arrived once).
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned G, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned arrived = atomicAdd(bar, 1u);
    if (arrived == G - 1) {
      bar[0] = 0u;
      __threadfence();
      atomicExch(bar + 1, gen + 1u);
    } else {
      while (ld_acquire_gpu(bar + 1) == gen) {
      }
    }
    __threadfence();
  }
  gen += 1u;
  __syncthreads();
}

// Per-CTA partial dots over the CTA's nr rows, thread per column j (rows
// ascending): out[v*stride + j] = sum_rr M[j*ldm + rr] * vec_v[rr].
template <typename T, int NV>
__device__ __noinline__ void lg_coldot(const T* __restrict__ M, int64_t ldm, int nr, int j0,
                                       int j1, const T* v0, const T* v1, T* out, int64_t stride) {
  for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
    const T* col = M + (int64_t)j * ldm;
    T a0 = T(0), a1 = T(0);
    int rr = 0;
    for (; rr + 4 <= nr; rr += 4) {
      T m[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) m[u] = col[rr + u];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a0 = fma(m[u], v0[rr + u], a0);
        if (NV > 1) a1 = fma(m[u], v1[rr + u], a1);
      }
    }
    for (; rr < nr; ++rr) {
      const T mv = col[rr];
      a0 = fma(mv, v0[rr], a0);
      if (NV > 1) a1 = fma(mv, v1[rr], a1);
    }
    out[j] = a0;
    if (NV > 1) out[stride + j] = a1;
  }
}

// Reduce-scatter: for entries e in [e0, e1) of the per-CTA partial arrays
// part[g*pstride + e], g < G: final[e] = sum over g (kLgSub interleaved
// ascending chains, combined in ascending chain order).
template <typename T>
__device__ __noinline__ void lg_reduce_entries(const T* part, int64_t pstride, int G, int e0,
                                               int e1, T* fin, T* red) {
  const int sub = threadIdx.x % kLgSub, slot = threadIdx.x / kLgSub;
  constexpr int kSlots = kLgThreads / kLgSub;
  for (int eb = e0; eb < e1; eb += kSlots) {
    const int e = eb + slot;
    T acc = T(0);
    if (e < e1)
      for (int g = sub; g < G; g += kLgSub) acc += __ldcg(part + (int64_t)g * pstride + e);
    __syncthreads();
    red[slot * kLgSub + sub] = acc;
    __syncthreads();
    if (sub == 0 && e < e1) {
      T s = T(0);
      for (int q = 0; q < kLgSub; ++q) s += red[slot * kLgSub + q];
      fin[e] = s;
    }
  }
}

// out[rr] = sum_{j<nq} M[j*ldm + rr] * c[j] for the CTA's rows; threads split
// (row, column group), groups combined in ascending order.
template <typename T>
__device__ __noinline__ void lg_rows_gemv(const T* __restrict__ M, int64_t ldm, int nr, int nq,
                                          const T* c, T* out, T* red) {
  const int ngrp = blockDim.x / nr;  // nr <= 64 guaranteed by the host
  const int rr = threadIdx.x % nr, grp = threadIdx.x / nr;
  T acc = T(0);
  if (grp < ngrp)
    for (int j = grp; j < nq; j += ngrp) acc = fma(M[(int64_t)j * ldm + rr], c[j], acc);
  __syncthreads();
  if (grp < ngrp) red[grp * nr + rr] = acc;
  __syncthreads();
  if (threadIdx.x < nr) {
    T s = T(0);
    for (int q = 0; q < ngrp; ++q) s += red[q * nr + threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

// Upper-triangular rows: out[o-o0] = sum_{l=o}^{l1-1} M[l*ldm + o] * c[l] for
// o in [o0, o1); threads split (output, column group), combined in order.
template <typename T>
__device__ __noinline__ void lg_trmv_rows(const T* __restrict__ M, int64_t ldm, int o0, int o1,
                                          int l1, const T* c, T* out, T* red) {
  const int no = o1 - o0;
  if (no <= 0) return;
  const int per = blockDim.x / no;  // threads per output (no <= 64 guaranteed)
  const int ol = threadIdx.x / per, q = threadIdx.x % per;
  T acc = T(0);
  if (ol < no) {
    const int o = o0 + ol;
    for (int l = o + q; l < l1; l += per) acc = fma(M[(int64_t)l * ldm + o], c[l], acc);
  }
  __syncthreads();
  if (ol < no) red[ol * per + q] = acc;
  __syncthreads();
  if (threadIdx.x < no) {
    T s = T(0);
    for (int u = 0; u < per; ++u) s += red[threadIdx.x * per + u];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

template <typename T>
__device__ __noinline__ void lg_reduce_parts(const double* parts, int nparts, int k, int ra,
                                             int nr, double scale, T* v, double* red) {
  // canonical 8-chain order (sgs_common.cuh canon_sum), chains in parallel
  const int g = threadIdx.x / 64, rl = threadIdx.x % 64;
  double acc = 0.0;
  if (rl < nr)
    for (int q = g; q < nparts; q += kCanonG) acc += __ldcg(parts + (int64_t)q * k + ra + rl);
  __syncthreads();
  red[g * 64 + rl] = acc;
  __syncthreads();
  if (threadIdx.x < nr) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < kCanonG; ++q) t += red[q * 64 + threadIdx.x];
    v[threadIdx.x] = from_double<T>(scale * t);
  }
  __syncthreads();
}

template <typename T>
__device__ __forceinline__ T lg_local_sum(T x, T* red) { return block_sum(x, red); }

template <typename T>
__global__ void __launch_bounds__(kLgThreads, 1) ls_grid_kernel(sgs_ls_args a) {
  pdl_enter();
  const int G = gridDim.x, g = blockIdx.x;
  const int k = a.k, cap = a.cap;
  const int ra = (int)(((int64_t)g * k) / G);
  const int rb = (int)(((int64_t)(g + 1) * k) / G);
  const int nr = rb - ra;
  const int64_t code0 = *reinterpret_cast<volatile const int64_t*>(&a.st->code);
  double dmax = a.st->diag_max, dmin = a.st->diag_min;
  if (code0 != 0) return;  // uniform: no CTA writes st before the first barrier

  T* scr = reinterpret_cast<T*>(a.scratch);
  const int64_t sA = 2 * (int64_t)cap + 8;
  T* XA = scr;                          // G x sA   per-CTA partials (exchange 1)
  T* XF = XA + (int64_t)kLgMaxG * sA;   // sA       reduced entries
  T* XB = XF + sA;                      // G x 8    per-CTA partials (exchange 2)
  T* XR = XB + (int64_t)kLgMaxG * 8;    // G x sA   reorthogonalisation partials
  T* XG = XR + (int64_t)kLgMaxG * sA;   // sA       reduced reorthogonalisation entries
  unsigned* bar = reinterpret_cast<unsigned*>(XG + sA);
  unsigned gen = ld_acquire_gpu(bar + 1);

  __shared__ T vs[64], vt[64], vp[64], tmp[64];
  __shared__ T red[kLgThreads];
  __shared__ double dred[kLgThreads];
  extern __shared__ unsigned char smem_raw[];
  T* fe = reinterpret_cast<T*>(smem_raw);  // sA gathered entries
  T* cc = fe + sA;                         // cap coefficients
  T* zz = cc + cap;                        // cap z

  T* S = static_cast<T*>(a.S);
  T* P = static_cast<T*>(a.P);
  T* Tm = static_cast<T*>(a.Qs);
  T* Rinv = static_cast<T*>(a.Rinv);
  T* AL = static_cast<T*>(a.alpha);
  double* R = a.R;
  const bool fused = a.do_finalize && a.do_solve;
  long long* trc = (g == 0 && threadIdx.x == 0) ? a.trace : nullptr;
#define SGS_TR(ix) \
  do {             \
    if (trc) trc[ix] = clock64(); \
  } while (0)
  SGS_TR(0);
  auto slice = [&](int n, int& o0, int& o1) {
    o0 = (int)(((int64_t)g * n) / G);
    o1 = (int)(((int64_t)(g + 1) * n) / G);
  };
  T tp = T(0), alpha = T(0);

  if (a.do_finalize) {
    const int i = a.col_fin, nq = i;
    if (i == 0) {
      if (threadIdx.x < nr) vs[threadIdx.x] = P[ra + threadIdx.x];
      __syncthreads();
    } else {
      lg_reduce_parts<T>(a.s_partials, a.s_nparts, k, ra, nr, a.s_scale, vs, dred);
    }
    if (fused && threadIdx.x < nr) vp[threadIdx.x] = P[(int64_t)(i + 1) * k + ra + threadIdx.x];
    __syncthreads();
    SGS_TR(1);
    // ---- exchange 1: [ss', pp, T^T s' (nq), T^T p (nq)] ------------------------
    T* myA = XA + (int64_t)g * sA;
    T l0 = T(0), l1 = T(0);
    if (threadIdx.x == 0) {
      for (int rr = 0; rr < nr; ++rr) {
        const T pv = P[(int64_t)i * k + ra + rr];
        l0 = fma(vs[rr], vs[rr], l0);
        l1 = fma(pv, pv, l1);
      }
      myA[0] = l0;
      myA[1] = l1;
    }
    if (nq > 0) {
      if (fused) lg_coldot<T, 2>(Tm + ra, k, nr, 0, nq, vs, vp, myA + 2, cap);
      else lg_coldot<T, 1>(Tm + ra, k, nr, 0, nq, vs, nullptr, myA + 2, cap);
    }
    const int E = 2 + (fused ? 2 * cap : (nq > 0 ? cap : 0));
    grid_sync(bar, G, gen);  // B1
    SGS_TR(2);
    int e0, e1;
    slice(E, e0, e1);
    lg_reduce_entries<T>(XA, sA, G, e0, e1, XF, red);
    grid_sync(bar, G, gen);  // B2
    SGS_TR(3);
    for (int e = threadIdx.x; e < 2 + nq; e += blockDim.x) fe[e] = __ldcg(XF + e);
    if (fused)
      for (int j = threadIdx.x; j < nq; j += blockDim.x) fe[2 + cap + j] = __ldcg(XF + 2 + cap + j);
    __syncthreads();
    const double r_ii = (double)sqrt(fe[0]);
    const double tol = a.bf_ucrs * (double)sqrt(fe[1]);
    if (r_ii <= tol) {  // NaN compares false and propagates, as in numpy
      if (g == 0 && threadIdx.x == 0) {
        a.st->code = SGS_ST_BREAKDOWN;
        a.st->column = i + 1;
        a.st->r_ii = r_ii;
        a.st->tol = tol;
      }
      return;
    }
    const T rT = (T)r_ii;
    if (threadIdx.x < nr) {
      const T sv = vs[threadIdx.x] / rT;
      vs[threadIdx.x] = sv;
      S[(int64_t)i * k + ra + threadIdx.x] = sv;
    }
    for (int j = threadIdx.x; j < nq; j += blockDim.x) {
      const T aj = __ldcg(AL + j);
      const T cj = (fe[2 + j] / aj) / rT;  // (Qs^T s)_j
      fe[2 + j] = cj;
      cc[j] = cj / aj;                     // coefficient on the unnormalised column T_j
      if (fused) zz[j] = fe[2 + cap + j] / aj;  // (Qs^T p)_j
    }
    __syncthreads();
    if (nq > 0) {
      lg_rows_gemv<T>(Tm + ra, k, nr, nq, cc, tmp, red);
      if (threadIdx.x < nr) vt[threadIdx.x] = vs[threadIdx.x] - tmp[threadIdx.x];
    } else if (threadIdx.x < nr) {
      vt[threadIdx.x] = vs[threadIdx.x];
    }
    __syncthreads();
    if (threadIdx.x < nr) Tm[(int64_t)i * k + ra + threadIdx.x] = vt[threadIdx.x];
    __syncthreads();
    SGS_TR(4);
    // ---- exchange 2: ||t||^2 and t^T p (same per-CTA dot as lg_coldot) -----------
    T* myB = XB + (int64_t)g * 8;
    if (threadIdx.x == 0) {
      T lt = T(0);
      for (int rr = 0; rr < nr; ++rr) lt = fma(vt[rr], vt[rr], lt);
      myB[0] = lt;
    }
    if (fused) lg_coldot<T, 1>(Tm + ra, k, nr, i, i + 1, vp, nullptr, myB + 1 - i, 0);
    grid_sync(bar, G, gen);  // B3
    SGS_TR(5);
    T tt = T(0);
    {
      // every CTA reduces the two scalars itself (ascending CTA order)
      if (threadIdx.x < 2) {
        T s = T(0);
        for (int q = 0; q < G; ++q) s += __ldcg(XB + (int64_t)q * 8 + threadIdx.x);
        red[threadIdx.x] = s;
      }
      __syncthreads();
      tt = red[0];
      tp = red[1];
      __syncthreads();
    }
    const T ss = fe[0] / (rT * rT);
    if (nq > 0 && tt < T(0.5) * ss) {
      // cancellation: a second classical Gram-Schmidt pass on t
      T* myR = XR + (int64_t)g * sA;
      lg_coldot<T, 1>(Tm + ra, k, nr, 0, nq, vt, nullptr, myR + 2, cap);
      grid_sync(bar, G, gen);
      slice(2 + nq, e0, e1);
      lg_reduce_entries<T>(XR, sA, G, e0, e1, XG, red);
      grid_sync(bar, G, gen);
      for (int j = threadIdx.x; j < nq; j += blockDim.x) {
        const T aj = __ldcg(AL + j);
        const T c2 = __ldcg(XG + 2 + j) / aj;
        fe[2 + j] = fe[2 + j] + c2;
        cc[j] = c2 / aj;
      }
      __syncthreads();
      lg_rows_gemv<T>(Tm + ra, k, nr, nq, cc, tmp, red);
      if (threadIdx.x < nr) {
        const T t2 = vt[threadIdx.x] - tmp[threadIdx.x];
        vt[threadIdx.x] = t2;
        Tm[(int64_t)i * k + ra + threadIdx.x] = t2;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        T lt = T(0);
        for (int rr = 0; rr < nr; ++rr) lt = fma(vt[rr], vt[rr], lt);
        myR[0] = lt;
      }
      if (fused) lg_coldot<T, 1>(Tm + ra, k, nr, i, i + 1, vp, nullptr, myR + 1 - i, 0);
      grid_sync(bar, G, gen);
      if (threadIdx.x < 2) {
        T s = T(0);
        for (int q = 0; q < G; ++q) s += __ldcg(XR + (int64_t)q * sA + threadIdx.x);
        red[threadIdx.x] = s;
      }
      __syncthreads();
      tt = red[0];
      tp = red[1];
      __syncthreads();
    }
    alpha = sqrt(tt);
    // R_S^{-1} column i on this CTA's slice of [0, i+1)
    int u0, u1;
    slice(i + 1, u0, u1);
    const int u1c = min(u1, nq);
    if (u0 < u1c) {
      lg_trmv_rows<T>(Rinv, cap, u0, u1c, nq, fe + 2, tmp, red);
      if (threadIdx.x < u1c - u0)
        Rinv[(int64_t)i * cap + u0 + threadIdx.x] = alpha > T(0) ? -tmp[threadIdx.x] / alpha : T(0);
    }
    if (threadIdx.x == 0 && u0 <= i && i < u1)
      Rinv[(int64_t)i * cap + i] = alpha > T(0) ? T(1) / alpha : T(0);
    if (g == 0 && threadIdx.x == 0) {
      AL[i] = alpha;
      R[(int64_t)i * cap + i] = r_ii;
    }
    const double ad = (double)alpha;
    if (i == 0) { dmax = ad; dmin = ad; }
    else { dmax = fmax(dmax, ad); dmin = fmin(dmin, ad); }
    if (g == 0 && threadIdx.x == 0) {
      a.st->diag_max = dmax;
      a.st->diag_min = dmin;
      a.st->ncols = i + 1;
      a.st->r_ii = r_ii;
    }
    __syncthreads();
    SGS_TR(6);
  }

  if (a.do_solve) {
    const int c = a.col_sol, nq = c;
    if (!fused) {
      if (a.p_partials != nullptr) {
        lg_reduce_parts<T>(a.p_partials, a.p_nparts, k, ra, nr, a.p_scale, vp, dred);
        if (threadIdx.x < nr) P[(int64_t)c * k + ra + threadIdx.x] = vp[threadIdx.x];
      } else if (threadIdx.x < nr) {
        vp[threadIdx.x] = P[(int64_t)c * k + ra + threadIdx.x];
      }
      __syncthreads();
    }
    if (dmin < 1e-8 * fmax(dmax, 1.0)) {  // gram_schmidt.py:186-189
      if (g == 0 && threadIdx.x == 0) {
        a.st->code = SGS_ST_RANK;
        a.st->column = c + 1;
      }
      return;
    }
    if (fused) {
      if (threadIdx.x == 0) zz[c - 1] = tp / alpha;
    } else {
      // entries laid out as in the fused exchange: T^T p at offset 2 + cap
      T* myA = XA + (int64_t)g * sA;
      lg_coldot<T, 1>(Tm + ra, k, nr, 0, nq, vp, nullptr, myA + 2 + cap, 0);
      grid_sync(bar, G, gen);
      int e0, e1;
      slice(nq, e0, e1);
      lg_reduce_entries<T>(XA + 2 + cap, sA, G, e0, e1, XF + 2 + cap, red);
      grid_sync(bar, G, gen);
      for (int j = threadIdx.x; j < nq; j += blockDim.x)
        zz[j] = __ldcg(XF + 2 + cap + j) / __ldcg(AL + j);
    }
    __syncthreads();
    SGS_TR(7);
    int o0, o1;
    slice(nq, o0, o1);
    lg_trmv_rows<T>(Rinv, cap, o0, o1, nq, zz, tmp, red);
    if (threadIdx.x < o1 - o0) {
      const int o = o0 + threadIdx.x;
      const T r = tmp[threadIdx.x];
      R[(int64_t)c * cap + o] = (double)r;
      if (a.coarse_dtype == SGS_F32) static_cast<float*>(a.r_crs)[o] = cvt<float>(r);
      else static_cast<double*>(a.r_crs)[o] = (double)r;
    }
    SGS_TR(8);
  }
#undef SGS_TR
}

int ls_grid_size(int k) {
  int gsz = (k + kLgMinRows - 1) / kLgMinRows;
  const int sms = sm_count();
  if (gsz > sms) gsz = sms;
  if (gsz > kLgMaxG) gsz = kLgMaxG;
  if (gsz < 1) gsz = 1;
  return gsz;
}

template <typename T>
int launch_ls_grid_t(const sgs_ls_args* a, cudaStream_t s) {
  const int G = ls_grid_size(a->k);
  const int RM = (a->k + G - 1) / G;
  if (RM > 64) {
    set_error("ls_grid: k=%d needs more than 64 rows per CTA", a->k);
    return SGS_EINVAL;
  }
  const size_t smem = (size_t)(2 * a->cap + 8 + 2 * a->cap) * sizeof(T);
  if (smem > 200 * 1024) {
    set_error("ls_grid: cap=%d too large", a->cap);
    return SGS_EINVAL;
  }
  auto kern = ls_grid_kernel<T>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return check_ex(launch_ex(kern, dim3(G), dim3(kLgThreads), smem, s, 1, *a), "ls_grid_kernel");
}

int launch_ls_grid(const sgs_ls_args* a, cudaStream_t s) {
  if (a->fine_dtype == SGS_F64) return launch_ls_grid_t<double>(a, s);
  return launch_ls_grid_t<float>(a, s);
}

int64_t ls_grid_scratch_elems(int cap) {
  const int64_t sA = 2 * (int64_t)cap + 8;
  return 2 * (int64_t)kLgMaxG * sA + 2 * sA + (int64_t)kLgMaxG * 8 + 16;
}

}  // namespace sgs
