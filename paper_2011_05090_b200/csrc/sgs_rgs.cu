// Randomized Gram-Schmidt column step on sm_100a.
//
// * rgs_update_kernel: the tall-skinny projection update of RgsState.push
//   step 3 (gram_schmidt.py:316-319), q' = cast_crs(w) - Q_{i-1} r_crs, in the
//   coarse format.  Q is column-major so every column is one coalesced
//   128-bit stream; each thread owns 16 bytes of rows and keeps 8 columns of
//   loads in flight.  The deferred step-7 normalisation of the previous
//   column (gram_schmidt.py:329) is folded into the same pass.
// * ls_step_kernel: the k-dimensional work of push (steps 1-2, 5-7 and the
//   least-squares append) as ONE launch of a thread-block cluster, rows of
//   the k-vectors partitioned over the CTAs, cluster barriers between the
//   dependent reductions.  The sketched least-squares problem is solved with
//   an incrementally maintained QR of S (orthonormal Qs by two-pass classical
//   Gram-Schmidt, explicit R_S^{-1}) instead of the reference's sequential
//   Householder reflector chain (_IncrementalHouseholderQR,
//   gram_schmidt.py:122-190): the same least-squares solution, backward
//   stable for the well-conditioned S that RGS maintains, but built from
//   parallel GEMV/TRMV passes instead of i dependent dot products.

#include <cooperative_groups.h>
#include "sgs_common.cuh"

namespace cg = cooperative_groups;

namespace sgs {

template <typename T> struct VecT;
template <> struct VecT<float> { using type = float4; static constexpr int N = 4; };
template <> struct VecT<double> { using type = double2; static constexpr int N = 2; };

template <typename T>
__device__ __forceinline__ void vload(const T* p, T* v) {
  using V = typename VecT<T>::type;
  const V x = *reinterpret_cast<const V*>(p);
  if constexpr (VecT<T>::N == 4) { v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w; }
  else { v[0] = x.x; v[1] = x.y; }
}
template <typename T>
__device__ __forceinline__ void vstore(T* p, const T* v) {
  using V = typename VecT<T>::type;
  V x;
  if constexpr (VecT<T>::N == 4) { x.x = v[0]; x.y = v[1]; x.z = v[2]; x.w = v[3]; }
  else { x.x = v[0]; x.y = v[1]; }
  *reinterpret_cast<V*>(p) = x;
}

template <typename TO, typename TI>
__device__ __forceinline__ TO cvt(TI x) {
  if constexpr (sizeof(TO) == sizeof(TI)) return (TO)x;
  else if constexpr (sizeof(TO) == 4) return __double2float_rn((double)x);
  else return (TO)x;
}

constexpr int kUpdThreads = 256;
constexpr int kUpdUnroll = 8;

// Q[:, i] = cast(w) - Q[:, :i] @ rc   (coarse arithmetic, FMA chain over j)
template <typename TQ, typename TW>
__global__ void __launch_bounds__(kUpdThreads)
rgs_update_kernel(TQ* __restrict__ Q, int64_t ldq, int64_t n, int i, const TW* __restrict__ w,
                  const TQ* __restrict__ rc, int normalize_prev, const double* __restrict__ R,
                  int64_t ldr, const sgs_status* st) {
  if (status_stopped(st)) return;
  constexpr int V = VecT<TQ>::N;
  extern __shared__ unsigned char smem_raw[];
  TQ* rs = reinterpret_cast<TQ*>(smem_raw);
  for (int j = threadIdx.x; j < i; j += blockDim.x) rs[j] = rc[j];
  __syncthreads();
  const int64_t row0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * V;
  if (row0 >= n) return;
  const bool full = row0 + V <= n;
  TQ acc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = TQ(0);
  const int nplain = normalize_prev ? i - 1 : i;
  if (full) {
    int j = 0;
    for (; j + kUpdUnroll <= nplain; j += kUpdUnroll) {
      TQ q[kUpdUnroll][V];
#pragma unroll
      for (int u = 0; u < kUpdUnroll; ++u) vload(Q + (int64_t)(j + u) * ldq + row0, q[u]);
#pragma unroll
      for (int u = 0; u < kUpdUnroll; ++u) {
        const TQ c = rs[j + u];
#pragma unroll
        for (int v = 0; v < V; ++v) acc[v] = fma(q[u][v], c, acc[v]);
      }
    }
    for (; j < nplain; ++j) {
      TQ q[V];
      vload(Q + (int64_t)j * ldq + row0, q);
      const TQ c = rs[j];
#pragma unroll
      for (int v = 0; v < V; ++v) acc[v] = fma(q[v], c, acc[v]);
    }
    if (normalize_prev) {
      const int j = i - 1;
      const double rjj = R[(int64_t)j * ldr + j];
      TQ q[V];
      TQ* col = Q + (int64_t)j * ldq + row0;
      vload(col, q);
#pragma unroll
      for (int v = 0; v < V; ++v) q[v] = cvt<TQ>((double)q[v] / rjj);
      vstore(col, q);
      const TQ c = rs[j];
#pragma unroll
      for (int v = 0; v < V; ++v) acc[v] = fma(q[v], c, acc[v]);
    }
    TQ out[V];
#pragma unroll
    for (int v = 0; v < V; ++v) out[v] = cvt<TQ>(w[row0 + v]) - acc[v];
    vstore(Q + (int64_t)i * ldq + row0, out);
  } else {
    const int nv = (int)(n - row0);
    for (int j = 0; j < nplain; ++j) {
      const TQ c = rs[j];
      for (int v = 0; v < nv; ++v) acc[v] = fma(Q[(int64_t)j * ldq + row0 + v], c, acc[v]);
    }
    if (normalize_prev) {
      const int j = i - 1;
      const double rjj = R[(int64_t)j * ldr + j];
      const TQ c = rs[j];
      for (int v = 0; v < nv; ++v) {
        TQ* p = Q + (int64_t)j * ldq + row0 + v;
        const TQ q = cvt<TQ>((double)*p / rjj);
        *p = q;
        acc[v] = fma(q, c, acc[v]);
      }
    }
    for (int v = 0; v < nv; ++v) Q[(int64_t)i * ldq + row0 + v] = cvt<TQ>(w[row0 + v]) - acc[v];
  }
}

template <typename TQ>
__global__ void normalize_column_kernel(TQ* __restrict__ Q, int64_t n, const double* rjj_ptr,
                                        const sgs_status* st) {
  if (status_stopped(st)) return;
  const double rjj = *rjj_ptr;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    Q[r] = cvt<TQ>((double)Q[r] / rjj);
}

// z = A[:, :ncols] (upcast to fp64) @ y
template <typename TA>
__global__ void __launch_bounds__(256)
gemv_f64_kernel(const TA* __restrict__ A, int64_t lda, int64_t n, int ncols,
                const double* __restrict__ y, double* __restrict__ z) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double acc = 0.0;
  int j = 0;
  for (; j + 4 <= ncols; j += 4) {
    double a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = (double)A[(int64_t)(j + u) * lda + r];
#pragma unroll
    for (int u = 0; u < 4; ++u) acc = fma(a[u], __ldg(y + j + u), acc);
  }
  for (; j < ncols; ++j) acc = fma((double)A[(int64_t)j * lda + r], __ldg(y + j), acc);
  z[r] = acc;
}

template <typename T>
__global__ void transpose_kernel(const T* __restrict__ src, int64_t lds, T* __restrict__ dst,
                                 int64_t ldd, int64_t rows, int64_t cols) {
  __shared__ T tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int q = threadIdx.y; q < 32; q += blockDim.y) {
    const int64_t r = r0 + q, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[q][threadIdx.x] = src[r * lds + c];
  }
  __syncthreads();
  for (int q = threadIdx.y; q < 32; q += blockDim.y) {
    const int64_t c = c0 + q, r = r0 + threadIdx.x;
    if (r < rows && c < cols) dst[c * ldd + r] = tile[threadIdx.x][q];
  }
}

// ===========================================================================
// Cluster least-squares step.
constexpr int kLsThreads = 512;
constexpr int kLsWarps = kLsThreads / 32;
constexpr int kLsMaxCluster = 16;
constexpr int kLsChunk = 256;  // outputs per pass of the 2-D matvec helper
constexpr int kLsRowsPerCta = 192;

static int g_ls_max_cluster = 0;

static int ls_cluster_size_host(int k) {
  if (g_ls_max_cluster == 0) {
    const char* env = getenv("SGS_LS_MAX_CLUSTER");
    int v = env ? atoi(env) : kLsMaxCluster;
    if (v < 1) v = 1;
    if (v > kLsMaxCluster) v = kLsMaxCluster;
    g_ls_max_cluster = v;
  }
  int cl = (k + kLsRowsPerCta - 1) / kLsRowsPerCta;
  if (cl < 1) cl = 1;
  if (cl > g_ls_max_cluster) cl = g_ls_max_cluster;
  return cl;
}

struct LsCtx {
  int rank, CL, ra, rb, nr, k, cap;
};

// GEMV-T over own rows: xpart[j] = sum_{rr<nr} M[j*ldm + rr] * v[rr], j < ncols.
// Warp per column (4 in flight), lanes over rows, fixed shuffle tree.
template <typename T>
__device__ void ls_gemvT_rows(const T* __restrict__ M, int64_t ldm, int nr, int ncols,
                              const T* v, T* __restrict__ xpart) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j0 = warp * 4; j0 < ncols; j0 += kLsWarps * 4) {
    T acc[4] = {T(0), T(0), T(0), T(0)};
    for (int rr = lane; rr < nr; rr += 32) {
      const T vr = v[rr];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (j0 + u < ncols) acc[u] = fma(M[(int64_t)(j0 + u) * ldm + rr], vr, acc[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const T s = warp_sum(acc[u]);
      if (lane == 0 && j0 + u < ncols) xpart[j0 + u] = s;
    }
  }
}

// out[o - o0] = sum_{l in [lstart(o), l1)} M[l*ldm + o] * v[l] for o in [o0, o1),
// lstart(o) = UPPER ? max(o, l0) : l0.  Warps split l (stride 16), lanes split o;
// the per-warp partial sums are combined in fixed warp order.
template <typename T, bool UPPER>
__device__ void ls_matvec(const T* __restrict__ M, int64_t ldm, int o0, int o1, int l0, int l1,
                          const T* v, T* out, T* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int oc = o0; oc < o1; oc += kLsChunk) {
    const int ocn = min(kLsChunk, o1 - oc);
    T acc[kLsChunk / 32];
#pragma unroll
    for (int q = 0; q < kLsChunk / 32; ++q) acc[q] = T(0);
    for (int l = l0 + warp; l < l1; l += kLsWarps) {
      const T vl = v[l];
      const T* col = M + (int64_t)l * ldm;
#pragma unroll
      for (int q = 0; q < kLsChunk / 32; ++q) {
        const int ol = lane + 32 * q;
        const int o = oc + ol;
        if (ol < ocn && (!UPPER || l >= o)) acc[q] = fma(col[o], vl, acc[q]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kLsChunk / 32; ++q) red[warp * kLsChunk + lane + 32 * q] = acc[q];
    __syncthreads();
    for (int ol = threadIdx.x; ol < ocn; ol += blockDim.x) {
      T s = T(0);
      for (int w = 0; w < kLsWarps; ++w) s += red[w * kLsChunk + ol];
      out[oc - o0 + ol] = s;
    }
  }
  __syncthreads();
}

// c[j] = sum_{q<CL} xpart[q*cap + j] (fixed order), read through L2.
template <typename T>
__device__ void ls_gather(const T* xpart, int CL, int cap, int ncols, T* c) {
  for (int j = threadIdx.x; j < ncols; j += blockDim.x) {
    T s = T(0);
    for (int q = 0; q < CL; ++q) s += __ldcg(xpart + (int64_t)q * cap + j);
    c[j] = s;
  }
  __syncthreads();
}

template <typename T>
__device__ T ls_cluster_sum(T local, T* slot, int rank, int CL, T* red, cg::cluster_group& cl) {
  const T b = block_sum(local, red);
  if (threadIdx.x == 0) slot[rank] = b;
  cl.sync();
  T s = T(0);
  for (int q = 0; q < CL; ++q) s += __ldcg(slot + q);
  return s;
}

template <typename T>
__device__ __forceinline__ T ld_fine(const void* p, int64_t idx) {
  return static_cast<const T*>(p)[idx];
}

template <typename T>
__global__ void __launch_bounds__(kLsThreads, 1) ls_step_kernel(sgs_ls_args a) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int CL = (int)cl.num_blocks();
  const int k = a.k, cap = a.cap;
  const int ra = (int)(((int64_t)rank * k) / CL);
  const int rb = (int)(((int64_t)(rank + 1) * k) / CL);
  const int nr = rb - ra;
  const int RM = (k + CL - 1) / CL;

  // all CTAs read the status before anyone can write it (first write follows
  // a cluster barrier), so every CTA takes the same branches.
  const int64_t code0 = *reinterpret_cast<volatile const int64_t*>(&a.st->code);
  double dmax = a.st->diag_max, dmin = a.st->diag_min;
  if (code0 != 0) return;

  extern __shared__ unsigned char smem_raw[];
  T* vs = reinterpret_cast<T*>(smem_raw);  // RM   s (row slice)
  T* vt = vs + RM;                         // RM   t
  T* vp = vt + RM;                         // RM   p
  T* tmp = vp + RM;                        // RM   matvec output
  T* c1 = tmp + RM;                        // cap
  T* c2 = c1 + cap;                        // cap
  T* zc = c2 + cap;                        // cap
  T* red = zc + cap;                       // kLsWarps * kLsChunk

  T* scr = reinterpret_cast<T*>(a.scratch);
  T* X1 = scr;                                   // CL x cap
  T* X2 = X1 + (int64_t)kLsMaxCluster * cap;     // CL x cap
  T* XZ = X2 + (int64_t)kLsMaxCluster * cap;     // CL x cap
  T* N0 = XZ + (int64_t)kLsMaxCluster * cap;     // 16: sum s'^2
  T* N1 = N0 + kLsMaxCluster;                    // 16: sum p^2
  T* N2 = N1 + kLsMaxCluster;                    // 16: sum t^2

  T* S = static_cast<T*>(a.S);
  T* P = static_cast<T*>(a.P);
  T* Qs = static_cast<T*>(a.Qs);
  T* Rinv = static_cast<T*>(a.Rinv);
  double* R = a.R;
  // output slice of [0, nq) for the TRMVs
  auto oslice = [&](int nq, int& o0, int& o1) {
    o0 = (int)(((int64_t)rank * nq) / CL);
    o1 = (int)(((int64_t)(rank + 1) * nq) / CL);
  };

  if (a.do_finalize) {
    const int i = a.col_fin;
    T lss = T(0), lpp = T(0);
    for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) {
      const int r = ra + rr;
      T sp;
      const T pv = P[(int64_t)i * k + r];
      if (i == 0 || a.s_partials == nullptr) {
        sp = pv;  // column 1: s'_1 = p_1 (gram_schmidt.py:307-310)
      } else {
        double acc = 0.0;
        for (int q = 0; q < a.s_nparts; ++q) acc += a.s_partials[(int64_t)q * k + r];
        sp = from_double<T>(a.s_scale * acc);
      }
      vs[rr] = sp;
      lss = fma(sp, sp, lss);
      lpp = fma(pv, pv, lpp);
    }
    const T ss = ls_cluster_sum(lss, N0, rank, CL, red, cl);
    // N1 slot written after the N0 barrier: reuse the same barrier pattern
    const T pp = ls_cluster_sum(lpp, N1, rank, CL, red, cl);
    const double r_ii = (double)sqrt(ss);
    const double tol = a.bf_ucrs * (double)sqrt(pp);
    if (r_ii <= tol || !(r_ii == r_ii)) {
      if (rank == 0 && threadIdx.x == 0) {
        a.st->code = (r_ii <= tol) ? SGS_ST_BREAKDOWN : SGS_ST_NONFINITE;
        a.st->column = i + 1;
        a.st->r_ii = r_ii;
        a.st->tol = tol;
      }
      return;
    }
    const T rT = (T)r_ii;
    for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) {
      const T s = vs[rr] / rT;
      vs[rr] = s;
      S[(int64_t)i * k + ra + rr] = s;
    }
    __syncthreads();
    // ---- append s_i to the QR of S: two classical GS passes -----------------
    const int nq = i;
    if (nq > 0) {
      ls_gemvT_rows<T>(Qs + ra, k, nr, nq, vs, X1 + (int64_t)rank * cap);
      cl.sync();
      ls_gather<T>(X1, CL, cap, nq, c1);
      ls_matvec<T, false>(Qs + ra, k, 0, nr, 0, nq, c1, tmp, red);
      for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) vt[rr] = vs[rr] - tmp[rr];
      __syncthreads();
      ls_gemvT_rows<T>(Qs + ra, k, nr, nq, vt, X2 + (int64_t)rank * cap);
      cl.sync();
      ls_gather<T>(X2, CL, cap, nq, c2);
      ls_matvec<T, false>(Qs + ra, k, 0, nr, 0, nq, c2, tmp, red);
      for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) vt[rr] = vt[rr] - tmp[rr];
      __syncthreads();
    } else {
      for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) vt[rr] = vs[rr];
      __syncthreads();
    }
    T ltt = T(0);
    for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) ltt = fma(vt[rr], vt[rr], ltt);
    const T tt = ls_cluster_sum(ltt, N2, rank, CL, red, cl);
    const T alpha = sqrt(tt);
    for (int rr = threadIdx.x; rr < nr; rr += blockDim.x)
      Qs[(int64_t)i * k + ra + rr] = alpha > T(0) ? vt[rr] / alpha : T(0);
    // Rinv[:i, i] = -Rinv[:i, :i] (c1 + c2) / alpha ; Rinv[i, i] = 1/alpha
    if (nq > 0) {
      for (int j = threadIdx.x; j < nq; j += blockDim.x) c1[j] = c1[j] + c2[j];
      __syncthreads();
      int o0, o1;
      oslice(nq, o0, o1);
      ls_matvec<T, true>(Rinv, cap, o0, o1, 0, nq, c1, tmp, red);
      for (int o = o0 + threadIdx.x; o < o1; o += blockDim.x)
        Rinv[(int64_t)i * cap + o] = alpha > T(0) ? -tmp[o - o0] / alpha : T(0);
    }
    if (rank == 0 && threadIdx.x == 0) {
      Rinv[(int64_t)i * cap + i] = alpha > T(0) ? T(1) / alpha : T(0);
      R[(int64_t)i * cap + i] = r_ii;
    }
    const double ad = (double)alpha;
    if (i == 0) { dmax = ad; dmin = ad; }
    else { dmax = fmax(dmax, ad); dmin = fmin(dmin, ad); }
    if (rank == 0 && threadIdx.x == 0) {
      a.st->diag_max = dmax;
      a.st->diag_min = dmin;
      a.st->ncols = i + 1;
      a.st->r_ii = r_ii;
    }
  }

  if (a.do_solve) {
    const int col = a.col_sol;
    const int nq = col;
    if (a.do_finalize) cl.sync();  // Qs[:, i] and Rinv[:, i] visible cluster-wide
    for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) {
      const int r = ra + rr;
      T pv;
      if (a.p_partials != nullptr) {
        double acc = 0.0;
        for (int q = 0; q < a.p_nparts; ++q) acc += a.p_partials[(int64_t)q * k + r];
        pv = from_double<T>(a.p_scale * acc);
        P[(int64_t)col * k + r] = pv;
      } else {
        pv = P[(int64_t)col * k + r];
      }
      vp[rr] = pv;
    }
    __syncthreads();
    if (nq > 0) {
      // rank check of the sketched basis (gram_schmidt.py:186-189)
      if (dmin < 1e-8 * fmax(dmax, 1.0)) {
        if (rank == 0 && threadIdx.x == 0) {
          a.st->code = SGS_ST_RANK;
          a.st->column = col + 1;
        }
        return;
      }
      ls_gemvT_rows<T>(Qs + ra, k, nr, nq, vp, XZ + (int64_t)rank * cap);
      cl.sync();
      ls_gather<T>(XZ, CL, cap, nq, zc);
      int o0, o1;
      oslice(nq, o0, o1);
      ls_matvec<T, true>(Rinv, cap, o0, o1, 0, nq, zc, tmp, red);
      for (int o = o0 + threadIdx.x; o < o1; o += blockDim.x) {
        const T r = tmp[o - o0];
        R[(int64_t)col * cap + o] = (double)r;
        if (a.coarse_dtype == SGS_F32) static_cast<float*>(a.r_crs)[o] = cvt<float>(r);
        else static_cast<double*>(a.r_crs)[o] = (double)r;
      }
    }
  }
}

static size_t ls_smem_bytes(int k, int cap, int CL, size_t esize) {
  const int RM = (k + CL - 1) / CL;
  return (size_t)(4 * RM + 3 * cap + kLsWarps * kLsChunk + 8) * esize;
}

template <typename T>
static int launch_ls(const sgs_ls_args* a, cudaStream_t s) {
  const int CL = ls_cluster_size_host(a->k);
  const size_t smem = ls_smem_bytes(a->k, a->cap, CL, sizeof(T));
  auto kern = ls_step_kernel<T>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (CL > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL, 1, 1);
  cfg.blockDim = dim3(kLsThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, *a);
  if (e != cudaSuccess) {
    set_error("ls_step_kernel launch (cluster %d, smem %zu): %s", CL, smem, cudaGetErrorString(e));
    return SGS_ECUDA;
  }
  return check_launch("ls_step_kernel");
}

}  // namespace sgs

using namespace sgs;

extern "C" int sgs_rgs_update(void* Q, int q_dtype, int64_t ldq, int64_t n, int i, const void* w,
                              int w_dtype, const void* r_crs, int normalize_prev, const double* R,
                              int64_t ldr, const sgs_status* st, void* stream) {
  SGS_REQUIRE(Q && w, "update: null pointer");
  SGS_REQUIRE(i >= 0 && n >= 1 && ldq >= n && (ldq % 4) == 0, "update: bad sizes");
  SGS_REQUIRE(i == 0 || r_crs, "update: r_crs required for i > 0");
  SGS_REQUIRE(!normalize_prev || (i > 0 && R), "update: normalize_prev needs R and i > 0");
  SGS_REQUIRE(((uintptr_t)Q & 15) == 0, "update: Q must be 16-byte aligned");
  cudaStream_t s = as_stream(stream);
  const int V = q_dtype == SGS_F32 ? 4 : 2;
  const int64_t nthr = (n + V - 1) / V;
  const unsigned blocks = (unsigned)((nthr + kUpdThreads - 1) / kUpdThreads);
  const size_t smem = (size_t)(i > 0 ? i : 1) * (q_dtype == SGS_F32 ? 4 : 8);
#define SGS_UPD(TQ, TW)                                                                      \
  do {                                                                                       \
    auto kern = rgs_update_kernel<TQ, TW>;                                                   \
    if (smem > 48 * 1024)                                                                    \
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);    \
    kern<<<blocks, kUpdThreads, smem, s>>>(static_cast<TQ*>(Q), ldq, n, i,                   \
                                           static_cast<const TW*>(w),                        \
                                           static_cast<const TQ*>(r_crs), normalize_prev, R, \
                                           ldr, st);                                         \
  } while (0)
  if (q_dtype == SGS_F32 && w_dtype == SGS_F32) SGS_UPD(float, float);
  else if (q_dtype == SGS_F32 && w_dtype == SGS_F64) SGS_UPD(float, double);
  else if (q_dtype == SGS_F64 && w_dtype == SGS_F32) SGS_UPD(double, float);
  else if (q_dtype == SGS_F64 && w_dtype == SGS_F64) SGS_UPD(double, double);
  else {
    set_error("update: bad dtype");
    return SGS_EINVAL;
  }
#undef SGS_UPD
  return check_launch("rgs_update_kernel");
}

extern "C" int sgs_normalize_column(void* Q, int q_dtype, int64_t ldq, int64_t n, int col,
                                    const double* R, int64_t ldr, const sgs_status* st,
                                    void* stream) {
  SGS_REQUIRE(Q && R && col >= 0 && n >= 1, "normalize: bad args");
  cudaStream_t s = as_stream(stream);
  int64_t blocks = (n + 255) / 256;
  if (blocks > 4 * 148 * 4) blocks = 4 * 148 * 4;
  const double* rjj = R + (int64_t)col * ldr + col;
  if (q_dtype == SGS_F32)
    normalize_column_kernel<float><<<(unsigned)blocks, 256, 0, s>>>(
        static_cast<float*>(Q) + (int64_t)col * ldq, n, rjj, st);
  else
    normalize_column_kernel<double><<<(unsigned)blocks, 256, 0, s>>>(
        static_cast<double*>(Q) + (int64_t)col * ldq, n, rjj, st);
  return check_launch("normalize_column_kernel");
}

extern "C" int sgs_gemv_f64(const void* A, int a_dtype, int64_t lda, int64_t n, int ncols,
                            const double* y, double* z, void* stream) {
  SGS_REQUIRE(A && y && z && n >= 1 && ncols >= 0 && lda >= n, "gemv: bad args");
  cudaStream_t s = as_stream(stream);
  const unsigned blocks = (unsigned)((n + 255) / 256);
  if (a_dtype == SGS_F32)
    gemv_f64_kernel<float><<<blocks, 256, 0, s>>>(static_cast<const float*>(A), lda, n, ncols, y, z);
  else
    gemv_f64_kernel<double><<<blocks, 256, 0, s>>>(static_cast<const double*>(A), lda, n, ncols, y, z);
  return check_launch("gemv_f64_kernel");
}

extern "C" int sgs_transpose(const void* src, int64_t lds, void* dst, int64_t ldd, int64_t rows,
                             int64_t cols, int dtype, void* stream) {
  SGS_REQUIRE(src && dst && rows >= 1 && cols >= 1, "transpose: bad args");
  cudaStream_t s = as_stream(stream);
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  dim3 block(32, 8);
  if (dtype == SGS_F32)
    transpose_kernel<float><<<grid, block, 0, s>>>(static_cast<const float*>(src), lds,
                                                   static_cast<float*>(dst), ldd, rows, cols);
  else
    transpose_kernel<double><<<grid, block, 0, s>>>(static_cast<const double*>(src), lds,
                                                    static_cast<double*>(dst), ldd, rows, cols);
  return check_launch("transpose_kernel");
}

extern "C" int64_t sgs_ls_scratch_elems(int k, int cap) {
  (void)k;
  return 3 * (int64_t)kLsMaxCluster * cap + 4 * kLsMaxCluster;
}

extern "C" int sgs_ls_cluster_size(int k) { return ls_cluster_size_host(k); }

extern "C" int sgs_ls_step(const sgs_ls_args* a, void* stream) {
  SGS_REQUIRE(a && a->st && a->S && a->P && a->R && a->Qs && a->Rinv && a->scratch,
              "ls_step: null pointer");
  SGS_REQUIRE(a->k >= 1 && a->cap >= 1 && a->cap <= 8192 && a->k <= 65536, "ls_step: bad sizes");
  SGS_REQUIRE(!a->do_finalize || (a->col_fin >= 0 && a->col_fin < a->cap), "ls_step: bad col_fin");
  SGS_REQUIRE(!a->do_solve || (a->col_sol >= 1 && a->col_sol < a->cap && a->r_crs),
              "ls_step: bad col_sol");
  SGS_REQUIRE(!a->do_finalize || a->col_fin == 0 || a->s_partials, "ls_step: s_partials missing");
  SGS_REQUIRE(!(a->do_finalize && a->do_solve) || a->col_sol == a->col_fin + 1,
              "ls_step: fused solve must target the next column");
  cudaStream_t s = as_stream(stream);
  if (a->fine_dtype == SGS_F64) return launch_ls<double>(a, s);
  if (a->fine_dtype == SGS_F32) return launch_ls<float>(a, s);
  set_error("ls_step: bad fine dtype");
  return SGS_EINVAL;
}
