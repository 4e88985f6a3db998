// Two-stream coupling probe: primary A (16-CTA cluster, 200 KB smem, spins on a
// flag) on stream B; stream M waits for an event of A's launch, then launches
// secondary S (sets the flag).  Variants: 0 = launch-completion event,
// 1 = programmatic event with triggerAtBlockStart, 2 = no event (plain
// concurrency); each eager and captured into a CUDA graph.
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void primary(volatile int* f, int* out) {
  if (threadIdx.x == 0) {
    unsigned long long t0 = gt();
    while (f[0] == 0) { if (gt() - t0 > 1000000000ULL) { out[blockIdx.x] = -1; return; } }
    out[blockIdx.x] = 1;
  }
}
__global__ void secondary(volatile int* f) { if (threadIdx.x == 0 && blockIdx.x == 0) f[0] = 1; }

static cudaError_t run(int variant, cudaStream_t B, cudaStream_t M, int* f, int* out, cudaEvent_t ev, cudaEvent_t fork, cudaEvent_t join) {
  cudaEventRecord(fork, M);
  cudaStreamWaitEvent(B, fork, 0);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[3];
  cfg.gridDim = dim3(16); cfg.blockDim = dim3(512); cfg.stream = B; cfg.dynamicSmemBytes = 200 * 1024;
  int na = 0;
  at[na].id = cudaLaunchAttributeClusterDimension; at[na].val.clusterDim.x = 16; at[na].val.clusterDim.y = 1; at[na].val.clusterDim.z = 1; ++na;
  if (variant == 0) { at[na].id = cudaLaunchAttributeLaunchCompletionEvent; at[na].val.launchCompletionEvent.event = ev; at[na].val.launchCompletionEvent.flags = 0; ++na; }
  if (variant == 1) { at[na].id = cudaLaunchAttributeProgrammaticEvent; at[na].val.programmaticEvent.event = ev; at[na].val.programmaticEvent.flags = 0; at[na].val.programmaticEvent.triggerAtBlockStart = 1; ++na; }
  cfg.attrs = at; cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, primary, (volatile int*)f, out);
  if (e) return e;
  if (variant != 2) cudaStreamWaitEvent(M, ev, 0);
  secondary<<<8, 256, 0, M>>>(f);
  cudaEventRecord(join, B);
  cudaStreamWaitEvent(M, join, 0);
  return cudaGetLastError();
}

int main() {
  int *f, *out;
  cudaMalloc(&f, 64); cudaMalloc(&out, 64 * 4);
  cudaStream_t B, M; cudaStreamCreateWithFlags(&B, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&M, cudaStreamNonBlocking);
  cudaEvent_t ev, fork, join;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming); cudaEventCreateWithFlags(&fork, cudaEventDisableTiming); cudaEventCreateWithFlags(&join, cudaEventDisableTiming);
  cudaFuncSetAttribute(primary, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(primary, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  secondary<<<1, 32, 0, M>>>(f);  // load modules
  primary<<<1, 32>>>(f, out);
  cudaDeviceSynchronize();
  for (int variant = 0; variant < 3; ++variant) {
    for (int graph = 0; graph < 2; ++graph) {
      cudaMemset(f, 0, 64); cudaMemset(out, 0, 256); cudaDeviceSynchronize();
      cudaError_t e;
      if (!graph) {
        e = run(variant, B, M, f, out, ev, fork, join);
      } else {
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(M, cudaStreamCaptureModeGlobal);
        e = run(variant, B, M, f, out, ev, fork, join);
        cudaError_t ec = cudaStreamEndCapture(M, &g);
        if (e == cudaSuccess) e = ec;
        if (e == cudaSuccess) e = cudaGraphInstantiate(&ge, g, 0);
        if (e == cudaSuccess) e = cudaGraphLaunch(ge, M);
      }
      cudaError_t s = cudaStreamSynchronize(M);
      cudaError_t s2 = cudaDeviceSynchronize();
      int h[16]; cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
      printf("variant=%d graph=%d err=%s sync=%d,%d out0=%d\n", variant, graph, cudaGetErrorString(e), (int)s, (int)s2, h[0]);
      cudaGetLastError();
    }
  }
  return 0;
}
