// Can a PDL secondary run while its primary (persistent, spinning) is still
// resident?  Primary A waits for a flag that secondary B sets; variants: A as
// a 16-CTA cluster or single CTAs, with/without griddepcontrol.wait first,
// with a plain kernel before A.  Prints which variants completed (no timeout).
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void plain(int* f) { if (threadIdx.x == 0 && blockIdx.x == 0) f[1] = 0; }

__global__ void primary(volatile int* f, int do_wait, int* out) {
  if (do_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) {
    unsigned long long t0 = gt();
    while (f[0] == 0) { if (gt() - t0 > 1000000000ULL) { out[blockIdx.x] = -1; return; } }
    out[blockIdx.x] = 1;
  }
}
__global__ void secondary(volatile int* f) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) f[0] = 1;
}

int main() {
  int *f, *out;
  cudaMalloc(&f, 64); cudaMalloc(&out, 64 * 4);
  cudaStream_t s; cudaStreamCreate(&s);
  for (int variant = 0; variant < 8; ++variant) {
    const int clus = (variant & 1) ? 16 : 1, do_wait = (variant >> 1) & 1, pre = (variant >> 2) & 1;
    cudaMemset(f, 0, 64); cudaMemset(out, 0, 256); cudaDeviceSynchronize();
    if (pre) plain<<<1, 32, 0, s>>>(f);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[2];
    cfg.gridDim = dim3(16); cfg.blockDim = dim3(512); cfg.stream = s;
    cfg.dynamicSmemBytes = 200 * 1024;
    int na = 0;
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[na].val.programmaticStreamSerializationAllowed = 1; ++na;
    if (clus > 1) { at[na].id = cudaLaunchAttributeClusterDimension; at[na].val.clusterDim.x = clus; at[na].val.clusterDim.y = 1; at[na].val.clusterDim.z = 1; ++na; }
    cfg.attrs = at; cfg.numAttrs = na;
    cudaFuncSetAttribute(primary, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(primary, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaError_t e1 = cudaLaunchKernelEx(&cfg, primary, (volatile int*)f, do_wait, out);
    cudaLaunchConfig_t c2 = {};
    cudaLaunchAttribute a2[2];
    c2.gridDim = dim3(8); c2.blockDim = dim3(512); c2.stream = s;
    a2[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; a2[0].val.programmaticStreamSerializationAllowed = 1;
    a2[1].id = cudaLaunchAttributeClusterDimension; a2[1].val.clusterDim.x = 8; a2[1].val.clusterDim.y = 1; a2[1].val.clusterDim.z = 1;
    c2.attrs = a2; c2.numAttrs = 2;
    cudaError_t e2 = cudaLaunchKernelEx(&c2, secondary, (volatile int*)f);
    cudaError_t e3 = cudaStreamSynchronize(s);
    int h[16]; cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
    printf("cluster=%d wait=%d pre=%d launch=%d,%d sync=%d out0=%d (1 = overlapped, -1 = timeout)\n", clus, do_wait, pre, (int)e1, (int)e2, (int)e3, h[0]);
  }
  return 0;
}
