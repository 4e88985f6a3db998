// Shared helpers for the sm_100a kernels of the RGS / RGMRES hot path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>
#include <cstdarg>
#include <atomic>
#include <utility>

#include "../../include/sketchgs_b200.h"

namespace sgs {

// ---- error plumbing -------------------------------------------------------
void set_error(const char* fmt, ...);
extern std::atomic<uint64_t> g_launches;

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return SGS_ECUDA;
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return SGS_OK;
}

#define SGS_REQUIRE(cond, ...)            \
  do {                                    \
    if (!(cond)) {                        \
      ::sgs::set_error(__VA_ARGS__);      \
      return SGS_EINVAL;                  \
    }                                     \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kMaxSMs = 148;
int sm_count();

// ---- device-side checks (the checked build) ------------------------------------
// `make checked` compiles the library with -DSGS_DEVICE_CHECKS into
// _lib/libsketchgs_b200_checked.so (SGS_LIB_CHECKED=1 loads it): every
// SGS_DCHECK then tests an index / shared-memory bound inside the kernels and
// traps with its location on a violation - the stand-in for compute-sanitizer
// memcheck, which this GPU pool does not run.  Compiled out otherwise.
#ifdef SGS_DEVICE_CHECKS
#define SGS_DCHECK(cond)                                                              \
  do {                                                                                \
    if (!(cond)) {                                                                    \
      printf("SGS_DCHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,  \
             (int)blockIdx.x, (int)threadIdx.x, #cond);                               \
      __trap();                                                                       \
    }                                                                                 \
  } while (0)
#else
#define SGS_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

// bytes of dynamic shared memory this launch was given
__device__ __forceinline__ uint32_t dyn_smem_bytes() {
  uint32_t v;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(v));
  return v;
}
// byte offset of p from the start of the dynamic shared memory window
__device__ __forceinline__ uint32_t dyn_smem_offset(const void* p, const void* base) {
  return (uint32_t)(reinterpret_cast<const unsigned char*>(p) -
                    reinterpret_cast<const unsigned char*>(base));
}

// ---- device helpers ---------------------------------------------------------
// Kernels handed a status block return early once a code is set, so a host
// that enqueued ahead of a breakdown/convergence turns the tail into no-ops.
__device__ __forceinline__ bool status_stopped(const sgs_status* st) {
  if (st == nullptr) return false;
  return *reinterpret_cast<const volatile int64_t*>(&st->code) != 0;
}

template <typename T> struct Vec4;
template <> struct Vec4<float> { using type = float4; };

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum with a fixed reduction tree (deterministic for a fixed
// blockDim).  `red` must hold blockDim/32 elements.  Result valid in all
// threads.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  T t = T(0);
  for (int w = 0; w < nw; ++w) t += red[w];  // same order in every thread
  return t;
}

// Two block sums sharing one barrier pair; each value follows block_sum's
// order exactly.  `red` must hold 2 * blockDim/32 elements.
template <typename T>
__device__ __forceinline__ void block_sum2(T& a, T& b, T* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  __syncthreads();
  if (lane == 0) {
    red[warp] = a;
    red[nw + warp] = b;
  }
  __syncthreads();
  T ta = T(0), tb = T(0);
  for (int w = 0; w < nw; ++w) {
    ta += red[w];
    tb += red[nw + w];
  }
  a = ta;
  b = tb;
}

// ---- programmatic dependent launch (PDL) ---------------------------------------
// Every hot-loop kernel is launched with programmatic stream serialisation: it
// may be scheduled while its predecessor drains, waits here before touching
// any predecessor output, and immediately lets its own successor launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_enter() {
  pdl_wait();
  pdl_trigger();
}

bool pdl_enabled();

// Optional debug timeline (sgs_debug_timeline): per column 8 x u64 of
// %globaltimer stamps, written by the column and LS kernels when non-null.
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
unsigned long long* debug_timeline();
// row of the debug timeline for the current step (sgs_debug_timeline_col), NULL when off
unsigned long long* debug_timeline_row();

// cudaLaunchKernelEx wrapper: PDL attribute (when enabled) + optional cluster.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                             cudaStream_t s, int cluster, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cluster > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = cluster;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

inline int check_ex(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    cudaGetLastError();
    return SGS_ECUDA;
  }
  return check_launch(what);
}

// 4096-row SRHT tiles are summed in groups of tile_group(n_local) consecutive
// tiles into one partial k-vector: by one CTA in tile order (batches), or by
// a cluster of that many CTAs through DSMEM in rank order (one column, and
// the fused column kernel's epilogue) - the same bits either way, and the same
// group for every kernel that sketches a vector of that length.  Groups of 4
// for grids of up to 256 tiles: c1's column grid is then 62 clusters of 4
// instead of 31 of 8 and leaves a GPC free, so the 16-CTA LS cluster of the
// column is resident from the column kernel's start and its pre-wait part
// overlaps the Q stream (c1: 5800 -> 5928 columns/s on the same power-capped
// box class).  Larger (multi-wave) grids keep groups of 8: half the partials
// for the LS to reduce (c3's 512 tiles: the one-sync fp32 variant 3584 ->
// 3675 Arnoldi steps/s).
constexpr int kTileGroupMax = 8;
__host__ __device__ inline int tile_group(int64_t n_local) {
  const int64_t nt = (n_local + 4095) / 4096;
  return nt <= 256 ? 4 : 8;
}

// Device descriptor of a row-sharded state's peer exchange (sgs_peer_*):
// rank q's area holds, at fixed offsets, its generation counter, the receive
// slots recv[parity][source rank][k] (fp64) and the flags
// flags[parity][source rank][CTA of the LS cluster].
constexpr int kPeerMaxWorld = 8;
constexpr int kPeerMaxCl = 16;
struct sgs_peer_desc_dev {
  int world, rank, k, pad;
  unsigned char* area[kPeerMaxWorld];
};
__host__ __device__ inline int64_t peer_recv_off() { return 256; }
__host__ __device__ inline int64_t peer_flag_off(int world, int k) {
  return 256 + ((int64_t)2 * world * k * 8 + 255) / 256 * 256;
}
__host__ __device__ inline int64_t peer_area_bytes(int world, int k) {
  return peer_flag_off(world, k) + (int64_t)2 * world * kPeerMaxCl * 4;
}

// Canonical order for summing per-CTA partials (used by every consumer so
// that the same vector reduced by different kernels gives the same bits):
// eight interleaved ascending chains acc_g = sum_{p = g mod 8} x_p, then
// sum_g acc_g in ascending g.
constexpr int kCanonG = 8;
__device__ __forceinline__ double canon_sum(const double* x, int64_t stride, int nparts) {
  double acc[kCanonG];
#pragma unroll
  for (int g = 0; g < kCanonG; ++g) acc[g] = 0.0;
  int p = 0;
  for (; p + kCanonG <= nparts; p += kCanonG) {
#pragma unroll
    for (int g = 0; g < kCanonG; ++g) acc[g] += x[(int64_t)(p + g) * stride];
  }
#pragma unroll
  for (int g = 0; g < kCanonG; ++g)
    if (p + g < nparts) acc[g] += x[(int64_t)(p + g) * stride];
  double t = 0.0;
#pragma unroll
  for (int g = 0; g < kCanonG; ++g) t += acc[g];
  return t;
}

template <typename T> __device__ __forceinline__ T from_double(double x);
template <> __device__ __forceinline__ double from_double<double>(double x) { return x; }
template <> __device__ __forceinline__ float from_double<float>(double x) { return __double2float_rn(x); }

// Q_{i-1} r of the RGS update in the coarse dtype: for fp32 Q, fma chains over
// blocks of kAccBlock consecutive columns with the block sums added in order
// (a single fp32 chain over i columns doubles the rounding error of the
// reference's OpenBLAS sgemv, whose SIMD dot products split the sum: measured
// on the oracle at n = 2^18, m = 200 mixed, ||W - QR||/||W|| 2.4e-7 with one
// chain, 1.06e-7 with blocks of 16, 1.04e-7 with sgemv).  fp64 keeps one chain.
// SGS_ACC_TWO=0 keeps the single chain for fp32 too (A/B switch); the flag is
// a kernel argument computed by acc_two<TQ>() on the host.
constexpr int kAccBlock = 16;
bool acc_two_enabled();
template <typename TQ> inline int acc_two() { return (sizeof(TQ) == 4 && acc_two_enabled()) ? 1 : 0; }

template <typename T> struct VecT;
template <> struct VecT<float> { using type = float4; static constexpr int N = 4; };
template <> struct VecT<double> { using type = double2; static constexpr int N = 2; };

template <typename T>
__device__ __forceinline__ void vload(const T* p, T* v) {
  using V = typename VecT<T>::type;
  // streaming (evict-first) load: the 1 GB-per-column Q stream must not evict
  // the small, reused k-dimensional state (S, P, T, R_S^{-1}) from L2
  const V x = __ldcs(reinterpret_cast<const V*>(p));
  if constexpr (VecT<T>::N == 4) { v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w; }
  else { v[0] = x.x; v[1] = x.y; }
}
template <typename T>
__device__ __forceinline__ void vload_smem(const T* p, T* v) {
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

}  // namespace sgs
