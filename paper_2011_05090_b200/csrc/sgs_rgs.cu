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

constexpr int kUpdThreads = 256;
constexpr int kUpdUnroll = 8;

// Q[:, i] = cast(w) - Q[:, :i] @ rc   (coarse arithmetic: fma chains over blocks
// of kAccBlock columns, block sums added in order - the two-level sum of the
// fused column kernel, sgs_column.cu)
template <typename TQ, typename TW>
__global__ void __launch_bounds__(kUpdThreads)
rgs_update_kernel(TQ* __restrict__ Q, int64_t ldq, int64_t n, int i, const TW* __restrict__ w,
                  const TQ* __restrict__ rc, int normalize_prev, const double* __restrict__ R,
                  int64_t ldr, const sgs_status* st, int two) {
  pdl_enter();
  if (status_stopped(st)) return;
  constexpr int V = VecT<TQ>::N;
  extern __shared__ unsigned char smem_raw[];
  TQ* rs = reinterpret_cast<TQ*>(smem_raw);
  for (int j = threadIdx.x; j < i; j += blockDim.x) rs[j] = rc[j];
  __syncthreads();
  const int64_t row0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * V;
  if (row0 >= n) return;
  const bool full = row0 + V <= n;
  TQ acc[V], tot[V];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = tot[v] = TQ(0);
  auto fold = [&](int j) {
    if (sizeof(TQ) == 4 && two && ((j + 1) & (kAccBlock - 1)) == 0) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        tot[v] += acc[v];
        acc[v] = TQ(0);
      }
    }
  };
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
        fold(j + u);
      }
    }
    for (; j < nplain; ++j) {
      TQ q[V];
      vload(Q + (int64_t)j * ldq + row0, q);
      const TQ c = rs[j];
#pragma unroll
      for (int v = 0; v < V; ++v) acc[v] = fma(q[v], c, acc[v]);
      fold(j);
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
      fold(j);
    }
    TQ out[V];
#pragma unroll
    for (int v = 0; v < V; ++v) out[v] = cvt<TQ>(__ldcs(w + row0 + v)) - (tot[v] + acc[v]);
    vstore(Q + (int64_t)i * ldq + row0, out);
  } else {
    const int nv = (int)(n - row0);
    for (int j = 0; j < nplain; ++j) {
      const TQ c = rs[j];
      for (int v = 0; v < nv; ++v) acc[v] = fma(Q[(int64_t)j * ldq + row0 + v], c, acc[v]);
      fold(j);
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
      fold(j);
    }
    for (int v = 0; v < nv; ++v)
      Q[(int64_t)i * ldq + row0 + v] = cvt<TQ>(w[row0 + v]) - (tot[v] + acc[v]);
  }
}

template <typename TQ>
__global__ void normalize_column_kernel(TQ* __restrict__ Q, int64_t n, const double* rjj_ptr,
                                        const sgs_status* st) {
  pdl_enter();
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
// Cluster least-squares step (v3).
//
// Rows of every k-vector are split over the CTAs of one cluster (<= 16).  The
// orthogonal factor of S is kept UNNORMALISED, T = Qs diag(alpha), with the
// norms alpha in a device vector, so that everything the fused
// finalize(i) + solve(i+1) launch needs crosses the cluster in two exchanges:
//   #1  ||s'||^2, ||p_i||^2, T^T s', T^T p_{i+1}          (s' = Theta q'_i)
//   #2  ||t||^2, t^T p_{i+1}                               (t = s - Qs Qs^T s)
// (r_ii scales the first exchange afterwards: Qs^T s = (T^T s' / alpha) / r_ii).
// A second Gram-Schmidt pass runs only when ||t||^2 < ||s||^2 / 2.  Each
// column dot is computed by one fixed lane/shuffle pattern and summed over
// the CTAs in rank order, whichever launch computes it, so streaming push and
// the batched factorisation agree bit for bit.
constexpr int kLsThreads = 512;
constexpr int kLsWarps = kLsThreads / 32;
constexpr int kLsMaxCluster = 16;
// Rows of the k-vectors per CTA: the cluster is ceil(k / 64) CTAs, at most 16
// (SGS_LS_ROWS overrides).  Measured at k = 600 (c0 columns/s; c3 one-sync fp32
// Arnoldi steps/s): 96 rows (7 CTAs) 9172 / 3763, 64 (10 CTAs) 9290 / 3782, 48
// (13) 9299 / 3693, 38 (16) 9322 / 3661 - a larger cluster shortens the LS
// launch but takes SMs from the column grid it overlaps with.
constexpr int kLsRowsPerCta = 64;
constexpr int kLsChunk = 128;  // rows / outputs per pass of the 2-D helpers (4 per lane)
constexpr int kLsCpw = 8;      // columns in flight per warp

static int g_ls_max_cluster = 0;

static int ls_cluster_size_host(int k) {
  if (g_ls_max_cluster == 0) {
    const char* env = getenv("SGS_LS_MAX_CLUSTER");
    int v = env ? atoi(env) : kLsMaxCluster;
    if (v < 1) v = 1;
    if (v > kLsMaxCluster) v = kLsMaxCluster;
    g_ls_max_cluster = v;
  }
  static const int rows_per_cta = [] {
    const char* e = getenv("SGS_LS_ROWS");
    const int v = e ? atoi(e) : kLsRowsPerCta;
    return v >= 8 ? v : kLsRowsPerCta;
  }();
  int cl = (k + rows_per_cta - 1) / rows_per_cta;
  if (cl < 1) cl = 1;
  if (cl > g_ls_max_cluster) cl = g_ls_max_cluster;
  return cl;
}

// Transposed butterfly: V values per lane in, the sum over the warp of value
// index (lane / (32 / V)) out (pairwise sums are commutative, so the result is
// independent of which lane of a pair adds).  V <= 32, power of two.
template <typename T, int V>
__device__ __forceinline__ T warp_multi_reduce(T (&a)[V], int lane) {
  int n = V;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    if (n > 1) {
      const bool hi = (lane & off) != 0;
#pragma unroll
      for (int q = 0; q < V / 2; ++q) {
        if (q < n / 2) {
          const T send = hi ? a[q] : a[q + n / 2];
          const T keep = hi ? a[q + n / 2] : a[q];
          a[q] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      n >>= 1;
    } else {
      a[0] += __shfl_xor_sync(0xffffffffu, a[0], off);
    }
  }
  return a[0];
}

// Per-CTA partial dots of NV vectors with columns [j0, j1) of M over the
// CTA's nr rows: o[j] = sum_rr M[j*ldm + rr] * v[rr].  Warp per column (8
// columns in flight), lanes stride the rows, fixed xor-shuffle tree.
// Column j of the CTA's row slice of T: rows cached in shared memory for
// j < ncache (prefetched while the predecessor kernel ran), global otherwise.
template <typename T>
struct ColSrc {
  const T* sq;   // smem cache, column j at sq + j*ldc
  int ldc;
  int ncache;
  const T* g;    // global T + ra, column j at g + j*ldg
  int64_t ldg;
  __device__ __forceinline__ const T* col(int j) const {
    return j < ncache ? sq + (int64_t)j * ldc : g + (int64_t)j * ldg;
  }
};

// Per-CTA partial dots of NV vectors with columns [j0, j1) over the CTA's nr
// rows: o[j] = sum_rr M(rr, j) * v[rr].  Warp per column (8 columns in
// flight), lanes stride the rows, one transposed butterfly for the 8 sums.
template <typename T, int NV>
__device__ __noinline__ void ls_coldot(ColSrc<T> M, int nr, int j0, int j1, const T* v0,
                                       const T* v1, T* __restrict__ o0, T* __restrict__ o1,
                                       int w0 = 0, int nw = kLsWarps) {
  // warps [w0, w0 + nw) share the columns (which warp takes a column does not
  // change its sum); the others return at once
  const int lane = threadIdx.x & 31, warp = (int)(threadIdx.x >> 5) - w0;
  if (warp < 0) return;
  for (int rc = 0; rc < nr; rc += kLsChunk) {  // rows in chunks of 128 (4 per lane)
    const int rn = min(kLsChunk, nr - rc);
    T x0[4], x1[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int rr = rc + lane + 32 * q;
      x0[q] = (lane + 32 * q < rn) ? v0[rr] : T(0);
      x1[q] = (NV > 1 && lane + 32 * q < rn) ? v1[rr] : T(0);
    }
    for (int jb = j0 + warp * kLsCpw; jb < j1; jb += nw * kLsCpw) {
      T mv[kLsCpw][4];
#pragma unroll
      for (int u = 0; u < kLsCpw; ++u) {
        const T* cp = M.col(min(jb + u, j1 - 1)) + rc + lane;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          mv[u][q] = (jb + u < j1 && lane + 32 * q < rn) ? cp[32 * q] : T(0);
      }
      // per-lane partial dots of the 8 (x NV) columns, then one transposed
      // butterfly that leaves each column's sum in a group of lanes
      T vals[kLsCpw * NV];
#pragma unroll
      for (int u = 0; u < kLsCpw; ++u) {
        T a0 = T(0), a1 = T(0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          a0 = fma(mv[u][q], x0[q], a0);
          if (NV > 1) a1 = fma(mv[u][q], x1[q], a1);
        }
        vals[u] = a0;
        if (NV > 1) vals[kLsCpw + u] = a1;
      }
      const T r = warp_multi_reduce<T, kLsCpw * NV>(vals, lane);
      constexpr int kGrp = 32 / (kLsCpw * NV);  // lanes holding the same sum
      if ((lane & (kGrp - 1)) == 0) {
        const int idx = lane / kGrp;
        const int u = idx % kLsCpw;
        if (jb + u < j1) {
          T* o = (idx < kLsCpw) ? o0 : o1;
          if (rc == 0) o[jb + u] = r;
          else o[jb + u] += r;  // rows beyond 128 per CTA: chunk sums in order
        }
      }
    }
    if (rc + kLsChunk < nr) __syncwarp();
  }
}

// out[rr] = sum_{l < l1} M(rr, l) * c[l] for the CTA's rows rr < nr (lanes own
// rows, warps take 8 columns at a time, warp partials combined in order).
template <typename T>
__device__ __noinline__ void ls_rows_gemv(ColSrc<T> M, int nr, int l1, const T* c, T* out,
                                          T* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int oc = 0; oc < nr; oc += kLsChunk) {
    const int on = min(kLsChunk, nr - oc);
    T acc[4] = {T(0), T(0), T(0), T(0)};
    for (int lb = warp * kLsCpw; lb < l1; lb += kLsWarps * kLsCpw) {
      T mv[kLsCpw][4];
#pragma unroll
      for (int u = 0; u < kLsCpw; ++u) {
        const int l = lb + u;
        const T* cp = M.col(min(l, l1 - 1)) + oc + lane;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          mv[u][q] = (l < l1 && lane + 32 * q < on) ? cp[32 * q] : T(0);
      }
#pragma unroll
      for (int u = 0; u < kLsCpw; ++u) {
        const T cl = (lb + u < l1) ? c[lb + u] : T(0);
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] = fma(mv[u][q], cl, acc[q]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) red[warp * kLsChunk + lane + 32 * q] = acc[q];
    __syncthreads();
    for (int ol = threadIdx.x; ol < on; ol += blockDim.x) {
      T s = T(0);
      for (int w = 0; w < kLsWarps; ++w) s += red[w * kLsChunk + ol];
      out[oc + ol] = s;
    }
  }
  __syncthreads();
}

// Upper-triangular row slice: out[o - o0] = sum_{l=o}^{l1-1} M[l*ldm + o] * c[l]
// for o in [o0, o1).  Lanes own outputs (1 or 4 each), warps take columns
// (16 or 8 at a time), warp partials combined in ascending warp order.
template <typename T, bool UPPER>
__device__ __noinline__ void ls_matvec(const T* __restrict__ M, int64_t ldm, int o0, int o1,
                                       int l1, const T* c, T* out, T* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (o1 - o0 <= 32) {
    // narrow slice: one output per lane, 16 columns in flight per warp
    constexpr int kC = 16;
    const int on = o1 - o0;
    const int lstart = UPPER ? o0 : 0;
    T acc = T(0);
    for (int lb = lstart + warp * kC; lb < l1; lb += kLsWarps * kC) {
      T mv[kC];
#pragma unroll
      for (int u = 0; u < kC; ++u) {
        const int l = lb + u;
        const bool ok = l < l1 && lane < on && (!UPPER || l >= o0 + lane);
        mv[u] = ok ? M[(int64_t)l * ldm + o0 + lane] : T(0);
      }
#pragma unroll
      for (int u = 0; u < kC; ++u) acc = fma(mv[u], (lb + u < l1) ? c[lb + u] : T(0), acc);
    }
    __syncthreads();
    red[warp * 32 + lane] = acc;
    __syncthreads();
    if (threadIdx.x < on) {
      T s = T(0);
      for (int w = 0; w < kLsWarps; ++w) s += red[w * 32 + threadIdx.x];
      out[threadIdx.x] = s;
    }
    __syncthreads();
    return;
  }
  for (int oc = o0; oc < o1; oc += kLsChunk) {
    const int on = min(kLsChunk, o1 - oc);
    const int lstart = UPPER ? oc : 0;
    T acc[4] = {T(0), T(0), T(0), T(0)};
    for (int lb = lstart + warp * kLsCpw; lb < l1; lb += kLsWarps * kLsCpw) {
      T mv[kLsCpw][4];
#pragma unroll
      for (int u = 0; u < kLsCpw; ++u) {
        const int l = lb + u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int ol = lane + 32 * q;
          const bool ok = l < l1 && ol < on && (!UPPER || l >= oc + ol);
          mv[u][q] = ok ? M[(int64_t)l * ldm + oc + ol] : T(0);
        }
      }
#pragma unroll
      for (int u = 0; u < kLsCpw; ++u) {
        const T cl = (lb + u < l1) ? c[lb + u] : T(0);
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] = fma(mv[u][q], cl, acc[q]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) red[warp * kLsChunk + lane + 32 * q] = acc[q];
    __syncthreads();
    for (int ol = threadIdx.x; ol < on; ol += blockDim.x) {
      T s = T(0);
      for (int w = 0; w < kLsWarps; ++w) s += red[w * kLsChunk + ol];
      out[oc - o0 + ol] = s;
    }
  }
  __syncthreads();
}

// c[j] = (sum_{q<CL} part[q*stride + j]) / div[j]  (ascending q), j in [j0, j1).
template <typename T>
__device__ __noinline__ void ls_gather(const T* part, int64_t stride, int CL, int j0, int j1,
                                       const T* div, T* c, T* div_keep = nullptr) {
  for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) {  // CL <= 16: all loads in flight
    T v[kLsMaxCluster];
    const T dj = div ? __ldcg(div + j) : T(1);
#pragma unroll
    for (int q = 0; q < kLsMaxCluster; ++q)
      v[q] = q < CL ? __ldcg(part + (int64_t)q * stride + j) : T(0);
    T s = T(0);
#pragma unroll
    for (int q = 0; q < kLsMaxCluster; ++q) if (q < CL) s += v[q];
    c[j] = div ? s / dj : s;
    if (div_keep) div_keep[j] = dj;  // a later phase reuses the divisor from shared memory
  }
}

// v[rr] = cast(scale * canon_sum(parts[:, ra+rr])) for the CTA's rows; the
// eight canonical chains run in parallel thread groups.
template <typename T>
__device__ __noinline__ void ls_reduce_parts(const double* parts, int nparts, int k, int ra,
                                             int nr, double scale, T* v, double* red) {
  // 8 groups x 64 threads; a thread carries the chains of two rows (rl and
  // rl + 64) and issues 8 terms of each before adding them, so a reduction
  // over many parts (296 from the dense column kernel) takes a few L2 round
  // trips instead of one per 4 terms.  Each chain still adds its parts in
  // ascending order from 0.0 and the 8 chains are summed in group order: the
  // canonical partial sum (canon_sum), bit for bit.
  const int g = threadIdx.x >> 6, rl = threadIdx.x & 63;
  for (int r0 = 0; r0 < nr; r0 += 128) {
    const int rr0 = r0 + rl, rr1 = r0 + 64 + rl;
    const bool ok0 = rr0 < nr, ok1 = rr1 < nr;
    const double* p0 = parts + ra + (ok0 ? rr0 : 0);
    const double* p1 = parts + ra + (ok1 ? rr1 : 0);
    double acc0 = 0.0, acc1 = 0.0;
    int q = g;
    for (; q + 7 * kCanonG < nparts; q += 8 * kCanonG) {
      double a[8], b[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a[u] = ok0 ? __ldcg(p0 + (int64_t)(q + u * kCanonG) * k) : 0.0;
        b[u] = ok1 ? __ldcg(p1 + (int64_t)(q + u * kCanonG) * k) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc0 += a[u];
        acc1 += b[u];
      }
    }
    {  // the < 8 remaining terms of each chain: all loads in flight, then added in order
      double a[8], b[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool in = q + u * kCanonG < nparts;
        a[u] = (ok0 && in) ? __ldcg(p0 + (int64_t)(q + u * kCanonG) * k) : 0.0;
        b[u] = (ok1 && in) ? __ldcg(p1 + (int64_t)(q + u * kCanonG) * k) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (q + u * kCanonG < nparts) {
          acc0 += a[u];
          acc1 += b[u];
        }
    }
    __syncthreads();
    red[g * 128 + rl] = acc0;
    red[g * 128 + 64 + rl] = acc1;
    __syncthreads();
    if (threadIdx.x < 128 && r0 + (int)threadIdx.x < nr) {
      double t = 0.0;
#pragma unroll
      for (int c = 0; c < kCanonG; ++c) t += red[c * 128 + threadIdx.x];
      v[r0 + threadIdx.x] = from_double<T>(scale * t);
    }
  }
  __syncthreads();
}
// s' of a row-sharded state summed across the ranks inside the LS launch
// (sgs_ls_args.peer): this CTA's rows of the local partials in the canonical
// order (scale 1), stored into every rank's receive slots
// recv[parity][this rank] over NVLink, flagged (release, system scope) with
// the epoch (generation, column); then the CTA waits for the same rows of
// every rank and adds them in rank order from 0.0.  Every rank therefore
// holds bit-identical s' (the replicated LS needs no broadcast), and for one
// rank it is the unsharded reduction's s' bit for bit.  Receive slots and
// flags alternate by column parity: a rank can run at most one column ahead
// of another (its next finalize waits for the other's flags).  Returns true
// when the factorisation stopped (status) or the wait timed out.
template <typename T>
__device__ __noinline__ bool ls_peer_sum(const sgs_peer_desc_dev* d, const double* parts,
                                         int nparts, int k, int ra, int nr, double scale, T* v,
                                         double* red, int col, int cta, sgs_status* st) {
  if constexpr (sizeof(T) != 8) {
    return true;  // the host enables the exchange for an fp64 LS only
  } else {
    __shared__ int stop;
    const int world = d->world, me = d->rank, par = col & 1;
    ls_reduce_parts<T>(parts, nparts, k, ra, nr, 1.0, v, red);  // local rows, exact sums
    const unsigned int gen =
        *reinterpret_cast<volatile const unsigned int*>(d->area[me]);
    const unsigned int epoch = gen * 8192u + (unsigned int)col;
    for (int q = 0; q < world; ++q) {
      double* dst = reinterpret_cast<double*>(d->area[q] + peer_recv_off()) +
                    ((int64_t)par * world + me) * k + ra;
      for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) dst[rr] = v[rr];
    }
    __syncthreads();  // the CTA's rows are stored; thread 0 publishes them
    if (threadIdx.x == 0) {
      stop = 0;
      // one fence for the CTA (cumulative over the barrier): system scope for
      // peers on other GPUs, GPU scope when the only "peer" is this GPU (a
      // system fence per thread measured ~8 % of a c1 step under PCIe traffic)
      if (world > 1) __threadfence_system();
      else __threadfence();
      for (int q = 0; q < world; ++q) {
        unsigned int* f = reinterpret_cast<unsigned int*>(d->area[q] + peer_flag_off(world, k)) +
                          ((int64_t)par * world + me) * kPeerMaxCl + cta;
        if (world > 1)
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
        else
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
      }
    }
    __syncthreads();
    if ((int)threadIdx.x < world) {
      const unsigned int* f = reinterpret_cast<const unsigned int*>(d->area[me] +
                                                                    peer_flag_off(world, k)) +
                              ((int64_t)par * world + threadIdx.x) * kPeerMaxCl + cta;
      const unsigned long long t0 = gtimer();
      for (;;) {
        unsigned int x;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(x) : "l"(f) : "memory");
        if (x == epoch) break;
        if (*reinterpret_cast<volatile const int64_t*>(&st->code) != 0) { stop = 1; break; }
        if (gtimer() - t0 > 4000000000ULL) {
          atomicCAS(reinterpret_cast<unsigned long long*>(&st->code), 0ULL,
                    (unsigned long long)SGS_ST_TIMEOUT);
          stop = 1;
          break;
        }
        __nanosleep(64);
      }
    }
    __syncthreads();
    if (stop) return true;
    const double* rcv = reinterpret_cast<const double*>(d->area[me] + peer_recv_off()) +
                        (int64_t)par * world * k + ra;
    for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) {
      double sacc = 0.0;
      for (int q = 0; q < world; ++q) sacc += __ldcg(rcv + (int64_t)q * k + rr);
      v[rr] = from_double<T>(scale * sacc);
    }
    __syncthreads();
    return false;
  }
}

// Two partial sets (s' and p' of a one-synchronisation launch) in one pass,
// all loads of a row in flight together; each chain sums in ls_reduce_parts'
// order, so the results are bit-identical to two separate calls.
template <typename T>
__device__ __noinline__ void ls_reduce_parts2(const double* pa, int na, double sa, T* va,
                                              const double* pb, int nb, double sb, T* vb,
                                              int k, int ra, int nr, double* red) {
  const int g = threadIdx.x >> 6, rl = threadIdx.x & 63;  // 8 groups x 64 rows
  const int nmax = max(na, nb);
  for (int r0 = 0; r0 < nr; r0 += 64) {
    double acc_a = 0.0, acc_b = 0.0;
    const int rr = r0 + rl;
    if (rr < nr) {
      const double* p = pa + ra + rr;
      const double* q = pb + ra + rr;
      for (int j0 = g; j0 < nmax; j0 += 8 * kCanonG) {  // 8 terms per chain in flight
        double x[8], y[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int j = j0 + u * kCanonG;
          x[u] = j < na ? __ldcg(p + (int64_t)j * k) : 0.0;
          y[u] = j < nb ? __ldcg(q + (int64_t)j * k) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int j = j0 + u * kCanonG;
          if (j < na) acc_a += x[u];
          if (j < nb) acc_b += y[u];
        }
      }
    }
    __syncthreads();
    red[g * 64 + rl] = acc_a;
    red[(kCanonG + g) * 64 + rl] = acc_b;
    __syncthreads();
    if (threadIdx.x < 128) {
      const int h = threadIdx.x >> 6, o = threadIdx.x & 63;
      if (r0 + o < nr) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < kCanonG; ++q) t += red[(h * kCanonG + q) * 64 + o];
        if (h == 0) va[r0 + o] = from_double<T>(sa * t);
        else vb[r0 + o] = from_double<T>(sb * t);
      }
    }
  }
  __syncthreads();
}

// block_sum / block_sum2 (sgs_common.cuh) for the LS kernel's fixed 16 warps:
// the same shuffle tree and the same ascending warp order, with the 16 warp
// sums loaded together instead of one dependent shared-memory load per term.
template <typename T>
__device__ __forceinline__ T ls_block_sum(T v, T* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  T r[kLsWarps];
#pragma unroll
  for (int w = 0; w < kLsWarps; ++w) r[w] = red[w];
  T t = T(0);
#pragma unroll
  for (int w = 0; w < kLsWarps; ++w) t += r[w];
  return t;
}
template <typename T>
__device__ __forceinline__ void ls_block_sum2(T& a, T& b, T* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  __syncthreads();
  if (lane == 0) {
    red[warp] = a;
    red[kLsWarps + warp] = b;
  }
  __syncthreads();
  T ra[kLsWarps], rb[kLsWarps];
#pragma unroll
  for (int w = 0; w < kLsWarps; ++w) {
    ra[w] = red[w];
    rb[w] = red[kLsWarps + w];
  }
  T ta = T(0), tb = T(0);
#pragma unroll
  for (int w = 0; w < kLsWarps; ++w) {
    ta += ra[w];
    tb += rb[w];
  }
  a = ta;
  b = tb;
}

// Cluster sum of one scalar per CTA from slots[q*stride] (ascending q).
template <typename T>
__device__ __forceinline__ T ls_slot_sum(const T* slots, int64_t stride, int CL) {
  T v[kLsMaxCluster];  // all loads in flight, summed in ascending q
#pragma unroll
  for (int q = 0; q < kLsMaxCluster; ++q) v[q] = q < CL ? __ldcg(slots + (int64_t)q * stride) : T(0);
  T s = T(0);
#pragma unroll
  for (int q = 0; q < kLsMaxCluster; ++q) if (q < CL) s += v[q];
  return s;
}

// Shared-memory carve-up of ls_step_kernel (16-byte aligned sub-arrays).
__host__ __device__ constexpr size_t ls_align16(size_t x) { return (x + 15) / 16 * 16; }
template <typename T>
struct LsSmem {
  T *vs, *vt, *vp, *tmp, *c1, *zc, *c2, *yv, *to, *red, *sq;
  size_t bytes;  // fixed part (before the cache)
  __host__ __device__ LsSmem(unsigned char* base, int RM, int cap) {
    size_t off = 0;
    auto take = [&](size_t n) {
      T* p = reinterpret_cast<T*>(base + off);
      off += ls_align16(n * sizeof(T));
      return p;
    };
    vs = take(RM); vt = take(RM); vp = take(RM); tmp = take(RM);
    c1 = take(cap); zc = take(cap); c2 = take(cap); yv = take(cap); to = take(cap);
    const size_t nred = (size_t)kLsWarps * kLsChunk;
    red = take(nred * sizeof(T) >= 512 * sizeof(double) ? nred : 512 * sizeof(double) / sizeof(T));
    sq = reinterpret_cast<T*>(base + off);
    bytes = off;
  }
};

// The deferred T column of the previous finalize (its own register budget:
// inlined, it pushed the LS kernel into spilling).  Loads that column's c1
// (and c2 = c1 / alpha) into shared memory and, when pend >= 0, forms
// T[:, pend] = S[:, pend] - T[:, :pend] c2 for this CTA's rows (the explicit
// path's arithmetic), also into the cache slot.  Ends with a block barrier.
template <typename T>
__device__ __forceinline__ void ls_deferred_column(const T* coef, int pend, int ncoef, const T* AL,
                                                const T* S, T* Tm, ColSrc<T> TS, T* sq, int RM,
                                                int ncache, int k, int ra, int nr, T* c1, T* c2,
                                                T* vt, T* tmp, T* red) {
  for (int j = threadIdx.x; j < ncoef; j += blockDim.x) {
    const T cj = __ldcg(coef + j);
    c1[j] = cj;                       // kept for a solve-only launch (identity)
    c2[j] = cj / __ldcg(AL + j);      // as the explicit path: coefficient on T_j
  }
  __syncthreads();
  if (pend < 0) return;
  for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) vt[rr] = S[(int64_t)pend * k + ra + rr];
  __syncthreads();
  if (pend > 0) ls_rows_gemv<T>(TS, nr, pend, c2, tmp, red);  // columns < pend only
  for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) {
    const T tv = pend > 0 ? vt[rr] - tmp[rr] : vt[rr];
    Tm[(int64_t)pend * k + ra + rr] = tv;
    if (pend < ncache) sq[(int64_t)pend * RM + rr] = tv;
  }
  __syncthreads();
}

// The gi earlier Givens rotations applied to h = rc[0..gi] by one warp (see
// ls_step_kernel): outputs to Tc[0..gi), the carry to Tc[gi].  The warp stages
// up to 320 rotations and h entries in buf (3 x 320 doubles of shared memory)
// with all loads in flight, lane 0 runs the dependent chain from there (its
// operand loads do not depend on the carry), and the warp stores the outputs.
__device__ __noinline__ void ls_givens_chain(const double* rc, const double* cs, const double* sn,
                                             double* Tc, int gi, double* buf) {
  constexpr int kB = 320;
  const int lane = threadIdx.x & 31;
  double* bc = buf;
  double* bs = buf + kB;
  double* bh = buf + 2 * kB;
  double carry = rc[0];
  for (int j0 = 0; j0 < gi; j0 += kB) {
    const int nb = min(kB, gi - j0);
    for (int j = lane; j < nb; j += 32) {
      bc[j] = cs[j0 + j];
      bs[j] = sn[j0 + j];
      bh[j] = rc[j0 + j + 1];
    }
    __syncwarp();
    if (lane == 0) {
#pragma unroll 8
      for (int j = 0; j < nb; ++j) {
        const double c = bc[j], s_ = bs[j], hn = bh[j];
        bc[j] = __dadd_rn(__dmul_rn(c, carry), __dmul_rn(s_, hn));
        carry = __dadd_rn(__dmul_rn(-s_, carry), __dmul_rn(c, hn));
      }
    }
    __syncwarp();
    for (int j = lane; j < nb; j += 32) Tc[j0 + j] = bc[j];
    __syncwarp();
  }
  if (lane == 0) Tc[gi] = carry;
}

// PLAIN / MODE select compiled-out variants of the same code.
// PLAIN: a launch without the one-synchronisation p' partials, the peer
// exchange and the Givens chain (plain RGS-QR on one GPU); those branches are
// compiled out, which shortens the code the post-wait path steps through.
template <typename T, bool PLAIN, int MODE>
__global__ void __launch_bounds__(kLsThreads, 1) ls_step_kernel(sgs_ls_args a) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int CL = (int)cl.num_blocks();
#define xsync() cl.sync()
  const int k = a.k, cap = a.cap;
  const int ra = (rank * k) / CL;  // k <= 65536, CL <= 16: int32 arithmetic
  const int rb = ((rank + 1) * k) / CL;
  const int nr = rb - ra;
  const int RM = (k + CL - 1) / CL;
  // MODE 1: the launch is known to finalize column i and solve for i + 1
  // (fused); 2: finalize only; 3: solve only; 0: whatever the arguments say
  constexpr bool SPEC = MODE != 0;  // a specialised variant: no stamps
  const bool do_fin = MODE == 1 || MODE == 2 || (MODE == 0 && a.do_finalize);
  const bool do_sol = MODE == 1 || MODE == 3 || (MODE == 0 && a.do_solve);
  const bool fused = do_fin && do_sol;
  // one-synchronisation Arnoldi: p'_{i+1} = Theta A q'_i
  // arrives as partials with s'_i, and p_{i+1} = p'_{i+1} / r_ii
  const bool lag = !PLAIN && fused && a.p_lag && a.p_partials != nullptr;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  LsSmem<T> L(smem_raw, RM, cap);
  // fixed arrays + the cache of ncache columns of T fit; the row slice fits RM
  SGS_DCHECK(CL >= 1 && CL <= kLsMaxCluster && nr >= 0 && nr <= RM);
  SGS_DCHECK(L.bytes + (size_t)a.cache_cols * RM * sizeof(T) <= dyn_smem_bytes());
  SGS_DCHECK(!do_fin || (a.col_fin >= 0 && a.col_fin < cap));
  SGS_DCHECK(!do_sol || (a.col_sol >= 1 && a.col_sol < cap));
  T* vs = L.vs;    // RM   s' -> s (own rows)
  T* vt = L.vt;    // RM   t
  T* vp = L.vp;    // RM   p
  T* tmp = L.tmp;  // RM
  T* c1 = L.c1;    // cap  Qs^T s
  T* zc = L.zc;    // cap  Qs^T p
  T* c2 = L.c2;    // cap
  T* yv = L.yv;    // cap  R_S^{-1}[:, :c-1] z (own slice)
  T* to = L.to;    // cap  TRMV outputs
  T* red = L.red;  // kLsWarps * kLsChunk, 16-byte aligned (also used as doubles)
  T* sq = L.sq;    // cache: own rows of T, RM per column
  double* dred = reinterpret_cast<double*>(red);
  __shared__ T bc[8];

  const int64_t sA = 2 * (int64_t)cap + 8;     // exchange stride per CTA
  T* scr = reinterpret_cast<T*>(a.scratch);
  T* XA = scr;                                  // CL x sA
  T* XB = XA + kLsMaxCluster * sA;              // CL x 8
  T* XR = XB + kLsMaxCluster * 8;               // CL x sA
  T* AL = static_cast<T*>(a.alpha);             // cap: column norms of T
  T* myA = XA + rank * sA;
  T* myB = XB + rank * 8;
  T* myR = XR + rank * sA;
  T* S = static_cast<T*>(a.S);
  T* P = static_cast<T*>(a.P);
  T* Tm = static_cast<T*>(a.Qs);  // unnormalised T
  T* Rinv = static_cast<T*>(a.Rinv);
  double* R = a.R;
  long long* trc = (!SPEC && rank == 0 && threadIdx.x == 0) ? a.trace : nullptr;
#define SGS_TR(ix) \
  do {             \
    if (trc) trc[ix] = clock64(); \
  } while (0)
  auto slice = [&](int n, int& o0, int& o1) {
    o0 = (rank * n) / CL;  // n <= 8192
    o1 = ((rank + 1) * n) / CL;
  };

  // ---- before the dependency wait -------------------------------------------------
  // Everything the LS state (T, R_S^{-1}, alpha, P, status) provides was written
  // by earlier launches that completed before the predecessor started; only the
  // sketch partials of q'_i come from the predecessor.  So the cache of this
  // CTA's rows of T and, in the fused QR path, the whole solve except the last
  // column's term run while the predecessor column kernel is still streaming Q.
  SGS_TR(0);
  if (!SPEC && a.timeline && rank == 0 && threadIdx.x == 0) a.timeline[6] = gtimer();
  const int64_t code0 = *reinterpret_cast<volatile const int64_t*>(&a.st->code);
  double dmax = a.st->diag_max, dmin = a.st->diag_min;
  // Progressive Givens update of GMRES step gi = col_fin - 1 (krylov.py:282-301),
  // folded into this launch (one-synchronisation Arnoldi): H[:, gi] = R[:gi+2,
  // col_fin].  Its first gi entries are the r of the previous launch's solve,
  // so the chain of the gi earlier rotations runs here, before the wait, on the
  // last warp of rank 0 (which sits out the cache fill below); only the new
  // rotation needs r_ii.  The warp loads 32 rotations at a time and every lane
  // runs the same chain from shuffled operands (same operations as
  // givens_update).  The carry waits in T[gi, gi] for thread 0 (bar.syncs
  // between), which overwrites it with the new rotation.
  const int gi = (!PLAIN && a.giv_on && do_fin) ? a.col_fin - 1 : -1;
  const bool giv_warp = gi >= 0 && rank == 0 && code0 == 0 && (threadIdx.x >> 5) == (int)(blockDim.x >> 5) - 1;
  if (giv_warp) ls_givens_chain(R + (int64_t)a.col_fin * cap, a.giv_cs, a.giv_sn,
                                 a.giv_T + (int64_t)gi * a.giv_ldt, gi, dred);
  // The previous finalize may have deferred its T column: form it now, while
  // the predecessor kernel streams (same arithmetic as the explicit path:
  // t = s - T[:, :pend] c2, rows of this CTA, from the shared-memory cache).
  // Idempotent, so a launch that stops early and leaves t_pend set only makes
  // the next one redo it.
  // t_pend[0]: column still to be formed; t_pend[1]: last column finalized on
  // the fast path (its c1 / s' are in t_coef) - kept when [0] is cleared
  const int pend = a.t_pend ? *reinterpret_cast<volatile const int*>(a.t_pend) : -1;
  const int last_fast = a.t_pend ? *reinterpret_cast<volatile const int*>(a.t_pend + 1) : -1;
  const int ncols_t = do_fin ? a.col_fin : a.col_sol;  // columns of T in use
  const int ncache = min(ncols_t, a.cache_cols);
  if (!giv_warp) {  // warp per column, 4 columns x 3 row groups of loads in flight per lane
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x >> 5) - ((gi >= 0 && rank == 0 && code0 == 0) ? 1 : 0);
    for (int rb0 = 0; rb0 < nr; rb0 += 96)
      for (int j0 = wid * 4; j0 < ncache; j0 += nw * 4) {
        T v[4][3];
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            const int j = j0 + c, rr = rb0 + lane + 32 * r;
            v[c][r] = (j < ncache && rr < nr) ? Tm[(int64_t)j * k + ra + rr] : T(0);
          }
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            const int j = j0 + c, rr = rb0 + lane + 32 * r;
            if (j < ncache && j != pend && rr < nr) sq[(int64_t)j * RM + rr] = v[c][r];
          }
      }
  }
  SGS_TR(11);
  const ColSrc<T> TS{sq, RM, ncache, Tm + ra, (int64_t)k};
  // a solve-only launch whose newest column was finalized on the fast path
  // evaluates z by the identity below and needs that column's c1 (even when
  // an earlier launch - e.g. a push that broke down - already formed T)
  const bool need_c1 = !do_fin && do_sol && last_fast >= 0 && last_fast == a.col_sol - 1;
  if ((pend >= 0 || need_c1) && code0 == 0)
    ls_deferred_column<T>(static_cast<const T*>(a.t_coef), pend, pend >= 0 ? pend : last_fast, AL,
                          S, Tm, TS, sq, RM, ncache, k, ra, nr, c1, c2, vt, tmp, red);
  __syncthreads();
  SGS_TR(12);
  int s0 = 0, s1 = 0;  // output slice of the solve: [0, c) for c = col_sol
  if (do_sol) slice(a.col_sol, s0, s1);
  if (fused && !lag && code0 == 0) {
    const int i = a.col_fin;  // solve for c = i + 1 uses T[:, :i] now, T[:, i] later
    for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) vp[rr] = P[(int64_t)(i + 1) * k + ra + rr];
    __syncthreads();
    if (i > 0) {
      ls_coldot<T, 1>(TS, nr, 0, i, vp, nullptr, myA + 8 + cap, nullptr);
      xsync();
      SGS_TR(13);
      ls_gather<T>(XA + 8 + cap, sA, CL, 0, i, AL, zc);
      __syncthreads();
      ls_matvec<T, true>(Rinv, cap, s0, s1, i, zc, yv, red);  // y = R_S^{-1}[:, :i] z[:i]
    } else {
      for (int o = s0 + threadIdx.x; o < s1; o += blockDim.x) yv[o - s0] = T(0);
      __syncthreads();
    }
  }
  if (do_fin && code0 == 0) {  // ||p_i||^2 over this CTA's rows: P is an input
    const int64_t pi = (int64_t)a.col_fin * k + ra;
    T l1 = T(0);
    for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) l1 = fma(P[pi + rr], P[pi + rr], l1);
    l1 = ls_block_sum(l1, red);
    if (threadIdx.x == 0) bc[6] = l1;
  }
  SGS_TR(1);
  unsigned long long* tl = SPEC ? nullptr : a.timeline;  // no stamps in the specialised variants
  if (tl && rank == 0 && threadIdx.x == 0) tl[3] = gtimer();
  pdl_enter();
  if (tl && rank == 0 && threadIdx.x == 0) tl[4] = gtimer();
  SGS_TR(2);
  if (code0 != 0) return;  // uniform: nobody writes st before a cluster barrier

  T tp = T(0), alpha = T(0);
  if (do_fin) {
    const int i = a.col_fin;
    const int nq = i;
    if (i == 0) {
      for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) vs[rr] = P[ra + rr];  // s'_1 = p_1
      if (lag) ls_reduce_parts<T>(a.p_partials, a.p_nparts, k, ra, nr, a.p_scale, vp, dred);
    } else if (lag) {  // s' and p' together
      ls_reduce_parts2<T>(a.s_partials, a.s_nparts, a.s_scale, vs, a.p_partials, a.p_nparts,
                          a.p_scale, vp, k, ra, nr, dred);
    } else if (!PLAIN && a.peer != nullptr) {  // s' summed across the ranks here (row-sharded state)
      if (ls_peer_sum<T>(static_cast<const sgs_peer_desc_dev*>(a.peer), a.s_partials, a.s_nparts,
                         k, ra, nr, a.s_scale, vs, dred, i, rank, a.st))
        return;  // uniform: every rank and CTA sees the same status / flags
    } else {
      ls_reduce_parts<T>(a.s_partials, a.s_nparts, k, ra, nr, a.s_scale, vs, dred);
    }
    __syncthreads();
    SGS_TR(3);
    // ---- exchange #1: ||s'||^2, ||p_i||^2, T^T s' --------------------------------
    const bool defer = a.t_pend != nullptr;
    if (nr <= 128) {
      // Up to 128 rows per CTA (k <= 2048 on 16 CTAs): warp 0 alone forms the
      // two sums while warps 1..15 start on the column dots - no block
      // barrier in this phase.  Lane l holds the values threads l, l + 32,
      // l + 64, l + 96 would in the block-wide sum, each group of 32 goes
      // through the same shuffle tree, and the four warp sums are added in
      // warp order from 0: block_sum's result bit for bit (its other twelve
      // terms are +0).
      if (threadIdx.x < 32) {
        T l0 = T(0), l2 = T(0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int rr = (int)threadIdx.x + 32 * q;
          const T sv = rr < nr ? vs[rr] : T(0);
          T a0 = fma(sv, sv, T(0));
          T a2 = (defer && fused && rr < nr) ? fma(sv, vp[rr], T(0)) : T(0);  // s'^T p_{i+1}
          a0 = warp_sum(a0);
          a2 = warp_sum(a2);
          l0 += a0;
          l2 += a2;
        }
        if (threadIdx.x == 0) { myA[0] = l0; myA[1] = bc[6]; myA[2] = l2; }  // bc[6]: ||p_i||^2
      }
      SGS_TR(14);
      if (nq > 0) {
        if (lag) ls_coldot<T, 2>(TS, nr, 0, nq, vs, vp, myA + 8, myA + 8 + cap, 1, kLsWarps - 1);
        else ls_coldot<T, 1>(TS, nr, 0, nq, vs, nullptr, myA + 8, nullptr, 1, kLsWarps - 1);
      }
    } else {
    T l0 = T(0), l2 = T(0);
    for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) {
      l0 = fma(vs[rr], vs[rr], l0);
      if (defer && fused) l2 = fma(vs[rr], vp[rr], l2);  // s'^T p_{i+1}
    }
    if (defer && fused) ls_block_sum2(l0, l2, red);
    else l0 = ls_block_sum(l0, red);
    if (threadIdx.x == 0) { myA[0] = l0; myA[1] = bc[6]; myA[2] = l2; }  // bc[6]: ||p_i||^2
    SGS_TR(14);
    if (nq > 0) {
      if (lag) ls_coldot<T, 2>(TS, nr, 0, nq, vs, vp, myA + 8, myA + 8 + cap);  // + T^T p'
      else ls_coldot<T, 1>(TS, nr, 0, nq, vs, nullptr, myA + 8, nullptr);
    }
    }
    SGS_TR(15);  // thread 0's share of the column dots done
    xsync();
    SGS_TR(4);
    if (threadIdx.x < 3) bc[threadIdx.x] = ls_slot_sum(XA + threadIdx.x, sA, CL);
    if (nq > 0) ls_gather<T>(XA + 8, sA, CL, 0, nq, AL, c1, to);  // T^T s' / alpha; to = alpha
    if (lag && nq > 0) ls_gather<T>(XA + 8 + cap, sA, CL, 0, nq, AL, zc);  // T^T p' / alpha
    __syncthreads();
    SGS_TR(5);
    const double r_ii = (double)sqrt(bc[0]);
    const double tol = a.bf_ucrs * (double)sqrt(bc[1]);
    if (__builtin_expect(r_ii <= tol, 0)) {  // NaN compares false and propagates, as in numpy (gram_schmidt.py:325)
      if (rank == 0 && threadIdx.x == 0) {
        a.st->code = SGS_ST_BREAKDOWN;
        a.st->column = i + 1;
        a.st->r_ii = r_ii;
        a.st->tol = tol;
      }
      return;
    }
    const T rT = (T)r_ii;
    T sp_dot = bc[2];  // s'^T p_{i+1}
    if (lag) {  // p_{i+1} = p'_{i+1} / r_ii; Q_s^T p and s'^T p follow linearly
      sp_dot = bc[2] / rT;
      for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) {
        const T pv = vp[rr] / rT;
        vp[rr] = pv;
        P[(int64_t)(i + 1) * k + ra + rr] = pv;
      }
      for (int j = threadIdx.x; j < nq; j += blockDim.x) zc[j] = zc[j] / rT;
      __syncthreads();
      if (nq > 0) {
        ls_matvec<T, true>(Rinv, cap, s0, s1, nq, zc, yv, red);  // y = R_S^{-1}[:, :i] z[:i]
      } else {
        for (int o = s0 + threadIdx.x; o < s1; o += blockDim.x) yv[o - s0] = T(0);
        __syncthreads();
      }
    }
    T* sprime = defer ? static_cast<T*>(a.t_coef) + cap : nullptr;
    for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) {
      if (sprime) sprime[ra + rr] = vs[rr];  // s', for a solve-only launch's identity
      const T sv = vs[rr] / rT;
      vs[rr] = sv;
      S[(int64_t)i * k + ra + rr] = sv;
    }
    // the fast path's two sums ride along: a thread squares the c1 entries it
    // has just scaled, in the order of the separate pass it replaces
    T acc_c = T(0), acc_p = T(0);
    for (int j = threadIdx.x; j < nq; j += blockDim.x) {
      const T cj = c1[j] / rT;       // (Qs^T s)_j
      c1[j] = cj;
      c2[j] = cj / to[j];            // coefficient on the unnormalised column T_j (to = alpha)
      if (defer) {
        acc_c = fma(cj, cj, acc_c);
        if (fused) acc_p = fma(cj, zc[j], acc_p);
      }
    }
    if (!defer) __syncthreads();     // (block_sum's barriers publish c1 / c2 otherwise)
    SGS_TR(6);
    // Fast path: Q_s = T diag(1/alpha) is orthonormal, so ||t||^2 = ||s||^2 -
    // sum_j c1_j^2 and t^T p = s^T p - sum_j c1_j zc_j (zc = Q_s^T p from before
    // the wait).  Every CTA evaluates them from identical gathered values in
    // the same order, so the branch is uniform across the cluster.  Without
    // cancellation the estimate is accurate to a few ulps and r is published
    // without forming t; with it (the reorthogonalisation case) the explicit
    // path below runs.
    bool explicit_t = true;
    T tt = T(0);
    if (defer) {
      if (fused) ls_block_sum2(acc_c, acc_p, red);  // one barrier pair, block_sum's order
      else acc_c = ls_block_sum(acc_c, red);
      const T ss0 = bc[0] / (rT * rT);
      const T tt_est = ss0 - acc_c;
      if (nq == 0 || tt_est >= T(0.5) * ss0) {
        explicit_t = false;
        tt = tt_est;
        if (fused) tp = sp_dot / rT - acc_p;
        if (rank == 0) {
          T* coef = static_cast<T*>(a.t_coef);
          for (int j = threadIdx.x; j < nq; j += blockDim.x) coef[j] = c1[j];
          if (threadIdx.x == 0) {
            a.t_pend[0] = i;
            a.t_pend[1] = i;
          }
        }
      }
    }
    if (__builtin_expect(explicit_t, 0)) {
    if (nq > 0) {
      ls_rows_gemv<T>(TS, nr, nq, c2, tmp, red);
      for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) vt[rr] = vs[rr] - tmp[rr];
    } else {
      for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) vt[rr] = vs[rr];
    }
    __syncthreads();
    SGS_TR(5);
    // ---- exchange #2: ||t||^2 and t^T p (dot with the stored column) ------------------
    for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) Tm[(int64_t)i * k + ra + rr] = vt[rr];
    T lt = T(0);
    for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) lt = fma(vt[rr], vt[rr], lt);
    lt = ls_block_sum(lt, red);  // its __syncthreads also publishes the T_i stores in the CTA
    if (threadIdx.x == 0) myB[0] = lt;
    const ColSrc<T> TG{sq, RM, 0, Tm + ra, (int64_t)k};
    if (fused) ls_coldot<T, 1>(TG, nr, i, i + 1, vp, nullptr, myB + 1 - i, nullptr);
    xsync();
    SGS_TR(6);
    if (threadIdx.x < 2) bc[2 + threadIdx.x] = ls_slot_sum(XB + threadIdx.x, 8, CL);
    __syncthreads();
    tt = bc[2];
    tp = bc[3];
    const T ss = bc[0] / (rT * rT);
    // binary32 LS (UNIFIED32): always the second pass ("twice is enough");
    // binary64: only on cancellation
    if (nq > 0 && (sizeof(T) == 4 || tt < T(0.5) * ss)) {
      // cancellation: second classical Gram-Schmidt pass on t
      ls_coldot<T, 1>(TS, nr, 0, nq, vt, nullptr, myR + 8, nullptr);
      xsync();
      ls_gather<T>(XR + 8, sA, CL, 0, nq, AL, c2);
      __syncthreads();
      for (int j = threadIdx.x; j < nq; j += blockDim.x) {
        c1[j] = c1[j] + c2[j];
        c2[j] = c2[j] / __ldcg(AL + j);
      }
      __syncthreads();
      ls_rows_gemv<T>(TS, nr, nq, c2, tmp, red);
      for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) {
        const T t2 = vt[rr] - tmp[rr];
        vt[rr] = t2;
        Tm[(int64_t)i * k + ra + rr] = t2;
      }
      T l2 = T(0);
      for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) l2 = fma(vt[rr], vt[rr], l2);
      l2 = ls_block_sum(l2, red);
      if (threadIdx.x == 0) myR[0] = l2;
      if (fused) ls_coldot<T, 1>(TG, nr, i, i + 1, vp, nullptr, myR + 1 - i, nullptr);
      xsync();
      if (threadIdx.x < 2) bc[4 + threadIdx.x] = ls_slot_sum(XR + threadIdx.x, sA, CL);
      __syncthreads();
      tt = bc[4];
      tp = bc[5];
    }
    if (defer && rank == 0 && threadIdx.x == 0) {  // T[:, i] stored, z by explicit dot
      a.t_pend[0] = -1;
      a.t_pend[1] = -1;
    }
    }  // explicit_t
    SGS_TR(7);
    alpha = sqrt(tt);
    // R_S^{-1} column i on this CTA's slice of [0, i+1): -R_S^{-1}[:i,:i] c1 / alpha
    int u0, u1;
    slice(i + 1, u0, u1);
    const int u1c = min(u1, nq);
    if (u0 < u1c) {
      ls_matvec<T, true>(Rinv, cap, u0, u1c, nq, c1, to, red);
      for (int o = u0 + threadIdx.x; o < u1c; o += blockDim.x)
        Rinv[(int64_t)i * cap + o] = alpha > T(0) ? -to[o - u0] / alpha : T(0);
    }
    if (threadIdx.x == 0 && u0 <= i && i < u1)
      Rinv[(int64_t)i * cap + i] = alpha > T(0) ? T(1) / alpha : T(0);
    if (rank == 0 && threadIdx.x == 0) {
      AL[i] = alpha;
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
      if (gi >= 0) {  // the new rotation (same operations as givens_update)
        const double beta = R[0];
        if (gi == 0) a.giv_g[0] = beta;
        double* Tc = a.giv_T + (int64_t)gi * a.giv_ldt;
        const double hi = Tc[gi], hn = r_ii;
        const double rr = hypot(hi, hn);
        double c, sv;
        if (rr == 0.0) { c = 1.0; sv = 0.0; }
        else { c = hi / rr; sv = hn / rr; }
        a.giv_cs[gi] = c;
        a.giv_sn[gi] = sv;
        Tc[gi] = rr;
        Tc[gi + 1] = 0.0;
        const double gg = a.giv_g[gi];
        a.giv_g[gi + 1] = __dmul_rn(-sv, gg);
        a.giv_g[gi] = __dmul_rn(c, gg);
        const double est = fabs(a.giv_g[gi + 1]) / beta;
        a.giv_hist[gi] = est;
        a.st->iters = gi + 1;
        if (a.giv_tol >= 0.0 && est <= a.giv_tol) {  // later launches see it and return
          a.st->code = SGS_ST_CONVERGED;
          a.st->column = gi + 1;
        }
      }
    }
    __syncthreads();
    SGS_TR(8);
  }

  if (do_sol) {
    const int c = a.col_sol;  // r = R_S^{-1}[:c,:c] z, z = Qs[:, :c]^T p
    // rank check of the sketched basis (gram_schmidt.py:186-189)
    if (dmin < 1e-8 * fmax(dmax, 1.0)) {
      if (rank == 0 && threadIdx.x == 0) {
        a.st->code = SGS_ST_RANK;
        a.st->column = c + 1;
      }
      return;
    }
    T zl;  // z[c-1]
    if (fused) {
      zl = tp / alpha;  // (T_{c-1}^T p) / alpha_{c-1}; y was formed before the wait
    } else {
      if (a.p_partials != nullptr) {
        ls_reduce_parts<T>(a.p_partials, a.p_nparts, k, ra, nr, a.p_scale, vp, dred);
        for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) P[(int64_t)c * k + ra + rr] = vp[rr];
      } else {
        for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) vp[rr] = P[(int64_t)c * k + ra + rr];
      }
      __syncthreads();
      // Newest column deferred by its finalize: z from the same identity and
      // arithmetic as the fused launch (t^T p = s'^T p / r_ii - sum_j c1_j zc_j),
      // so streaming push and batch factorisation stay bit-identical.
      // re-read (unchanged within a solve-only launch) instead of keeping a
      // register live across the whole kernel
      const int last_fast_c = a.t_pend ? *reinterpret_cast<volatile const int*>(a.t_pend + 1) : -1;
      const bool idz = last_fast_c >= 0 && last_fast_c == c - 1;
      if (idz) {
        const T* sprime = static_cast<const T*>(a.t_coef) + cap;
        T l2 = T(0);
        for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) l2 = fma(__ldcg(sprime + ra + rr), vp[rr], l2);
        l2 = ls_block_sum(l2, red);
        if (threadIdx.x == 0) myA[2] = l2;
      }
      ls_coldot<T, 1>(TS, nr, 0, c, vp, nullptr, myA + 8 + cap, nullptr);
      xsync();
      // every CTA has read t_pend (pre-wait) and formed its rows of it
      if (!do_fin && a.t_pend != nullptr && rank == 0 && threadIdx.x == 0) a.t_pend[0] = -1;
      ls_gather<T>(XA + 8 + cap, sA, CL, 0, c, AL, zc);
      if (idz && threadIdx.x == 0) bc[2] = ls_slot_sum(XA + 2, sA, CL);
      __syncthreads();
      ls_matvec<T, true>(Rinv, cap, s0, s1, c - 1, zc, yv, red);
      if (idz) {
        T acc_p = T(0);
        for (int j = threadIdx.x; j < c - 1; j += blockDim.x) acc_p = fma(c1[j], zc[j], acc_p);
        acc_p = ls_block_sum(acc_p, red);
        const T rTn = (T)R[(int64_t)(c - 1) * cap + (c - 1)];
        zl = (bc[2] / rTn - acc_p) / __ldcg(AL + (c - 1));
      } else {
        zl = zc[c - 1];
      }
    }
    SGS_TR(9);
    // r_o = y_o + R_S^{-1}[o, c-1] z[c-1]  (same two-term form on every path)
    for (int o = s0 + threadIdx.x; o < s1; o += blockDim.x) {
      const T r = fma(Rinv[(int64_t)(c - 1) * cap + o], zl, yv[o - s0]);
      R[(int64_t)c * cap + o] = (double)r;
      if (a.coarse_dtype == SGS_F32) static_cast<float*>(a.r_crs)[o] = cvt<float>(r);
      else static_cast<double*>(a.r_crs)[o] = (double)r;
    }
    SGS_TR(10);
  }
  if (tl && rank == 0 && threadIdx.x == 0) tl[5] = gtimer();
#undef SGS_TR
#undef xsync
}

template <typename T>
static size_t ls_smem_fixed(int k, int cap, int CL) {
  const int RM = (k + CL - 1) / CL;
  return LsSmem<T>(nullptr, RM, cap).bytes;
}
constexpr size_t kLsSmemMax = 227 * 1024;

template <typename T>
static int launch_ls(const sgs_ls_args* a, cudaStream_t s) {
  const int CL = ls_cluster_size_host(a->k);
  const size_t fixed = ls_smem_fixed<T>(a->k, a->cap, CL);
  if (fixed > kLsSmemMax) {
    set_error("ls_step: k=%d cap=%d needs %zu bytes of shared memory", a->k, a->cap, fixed);
    return SGS_EINVAL;
  }
  const int RM = (a->k + CL - 1) / CL;
  const int ncols_t = a->do_finalize ? a->col_fin : 0;  // solve-only: read T once, no cache
  int cache = (int)((kLsSmemMax - fixed) / ((size_t)RM * sizeof(T)));
  if (cache > ncols_t) cache = ncols_t;
  if (cache < 0) cache = 0;
  const size_t smem = fixed + (size_t)cache * RM * sizeof(T);
  sgs_ls_args aa = *a;
  aa.cache_cols = cache;
  {
    unsigned long long* tlb = debug_timeline();
    const int col = a->do_finalize ? a->col_fin : a->col_sol;
    aa.timeline = tlb ? tlb + (int64_t)col * 16 + (a->do_finalize ? 0 : 3) : nullptr;
  }
  // SGS_LS_PLAIN=0: always the full variant; 1: PLAIN but no MODE variants (A/B)
  static const int plain_lvl = [] {
    const char* e = getenv("SGS_LS_PLAIN");
    return e ? atoi(e) : 2;
  }();
  const bool plain =
      plain_lvl >= 1 && !(a->p_lag && a->p_partials) && a->peer == nullptr && !a->giv_on;
  const bool spec = plain_lvl >= 2 && a->trace == nullptr && aa.timeline == nullptr;
  const int mode = !spec ? 0 : (a->do_finalize && a->do_solve) ? 1 : a->do_finalize ? 2 : 3;
  void (*kern)(sgs_ls_args) = nullptr;
#define SGS_LS_PICK(P)                                                        \
  kern = mode == 1 ? ls_step_kernel<T, P, 1> : mode == 2 ? ls_step_kernel<T, P, 2> \
       : mode == 3 ? ls_step_kernel<T, P, 3> : ls_step_kernel<T, P, 0>
  if (plain) SGS_LS_PICK(true);
  else SGS_LS_PICK(false);
#undef SGS_LS_PICK
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (CL > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  return check_ex(launch_ex(kern, dim3(CL), dim3(kLsThreads), smem, s, CL, aa), "ls_step_kernel");
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
  cudaError_t err = cudaSuccess;
#define SGS_UPD(TQ, TW)                                                                      \
  do {                                                                                       \
    auto kern = rgs_update_kernel<TQ, TW>;                                                   \
    if (smem > 48 * 1024)                                                                    \
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);    \
    err = launch_ex(kern, dim3(blocks), dim3(kUpdThreads), smem, s, 1, static_cast<TQ*>(Q),   \
                    ldq, n, i, static_cast<const TW*>(w), static_cast<const TQ*>(r_crs),     \
                    normalize_prev, R, ldr, st, acc_two<TQ>());                              \
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
  return check_ex(err, "rgs_update_kernel");
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
    return check_ex(launch_ex(normalize_column_kernel<float>, dim3((unsigned)blocks), dim3(256), 0,
                              s, 1, static_cast<float*>(Q) + (int64_t)col * ldq, n, rjj, st),
                    "normalize_column_kernel");
  return check_ex(launch_ex(normalize_column_kernel<double>, dim3((unsigned)blocks), dim3(256), 0,
                            s, 1, static_cast<double*>(Q) + (int64_t)col * ldq, n, rjj, st),
                  "normalize_column_kernel");
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
  const int64_t sA = 2 * (int64_t)cap + 8;
  return 2 * kLsMaxCluster * sA + kLsMaxCluster * 8 + 64;
}

extern "C" int sgs_ls_cluster_size(int k) { return ls_cluster_size_host(k); }

extern "C" int sgs_ls_step(const sgs_ls_args* a, void* stream) {
  SGS_REQUIRE(a && a->st && a->S && a->P && a->R && a->Qs && a->Rinv && a->alpha && a->scratch,
              "ls_step: null pointer");
  SGS_REQUIRE(a->k >= 1 && a->cap >= 1 && a->cap <= 8192 && a->k <= 65536, "ls_step: bad sizes");
  SGS_REQUIRE(!a->do_finalize || (a->col_fin >= 0 && a->col_fin < a->cap), "ls_step: bad col_fin");
  SGS_REQUIRE(!a->do_solve || (a->col_sol >= 1 && a->col_sol < a->cap && a->r_crs),
              "ls_step: bad col_sol");
  SGS_REQUIRE(!a->do_finalize || a->col_fin == 0 || a->s_partials, "ls_step: s_partials missing");
  SGS_REQUIRE(!(a->do_finalize && a->do_solve) || a->col_sol == a->col_fin + 1,
              "ls_step: fused solve must target the next column");
  SGS_REQUIRE(!a->p_lag || (a->do_finalize && a->do_solve && a->p_partials),
              "ls_step: p_lag needs a fused finalize + solve with p partials");
  SGS_REQUIRE(!a->peer || (a->fine_dtype == SGS_F64 && !a->p_lag && ls_cluster_size_host(a->k) <= kPeerMaxCl),
              "ls_step: the peer exchange needs an fp64 LS (no p_lag)");
  SGS_REQUIRE(!a->giv_on || (a->do_finalize && a->col_fin >= 1 && a->giv_cs && a->giv_sn &&
                             a->giv_g && a->giv_T && a->giv_hist && a->giv_ldt >= a->col_fin + 1),
              "ls_step: giv_on needs a finalize of column >= 1 and the Givens arrays");
  cudaStream_t s = as_stream(stream);
  if (a->fine_dtype == SGS_F64) return launch_ls<double>(a, s);
  if (a->fine_dtype == SGS_F32) return launch_ls<float>(a, s);
  set_error("ls_step: bad fine dtype");
  return SGS_EINVAL;
}
