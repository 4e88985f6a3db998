// Shared helpers for the sm_100a kernels of the RGS / RGMRES hot path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>
#include <cstdarg>
#include <atomic>

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

template <typename T> __device__ __forceinline__ T from_double(double x);
template <> __device__ __forceinline__ double from_double<double>(double x) { return x; }
template <> __device__ __forceinline__ float from_double<float>(double x) { return __double2float_rn(x); }

}  // namespace sgs
