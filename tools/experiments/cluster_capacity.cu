// How many clusters of the column-kernel shape (512 threads, 64 regs, ~84 KB
// smem) and of the LS shape (512 threads, 128 regs, 227 KB) can be resident
// at once on this GPU (cudaOccupancyMaxActiveClusters), per cluster size.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(512, 2) colshape(float* p) { extern __shared__ float s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }
__global__ void __launch_bounds__(512, 1) lsshape(float* p) { extern __shared__ float s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }
__global__ void __launch_bounds__(256, 4) col256(float* p) { extern __shared__ float s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }
template <typename K>
void probe(const char* name, K kern, int threads, size_t smem) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64); cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a; a.id = cudaLaunchAttributeClusterDimension; a.val.clusterDim.x = cs; a.val.clusterDim.y = 1; a.val.clusterDim.z = 1;
    cfg.attrs = &a; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
    printf("%s smem=%zuKB cluster=%2d max_active_clusters=%d (%d CTAs) %s\n", name, smem / 1024, cs, n, n * cs, e ? cudaGetErrorString(e) : "");
  }
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("%s SMs=%d\n", p.name, p.multiProcessorCount);
  probe("column(512x2/SM)", colshape, 512, 84 * 1024);
  probe("ls(512x1/SM)", lsshape, 512, 227 * 1024);
  probe("col256(256x4/SM)", col256, 256, 50 * 1024);
  return 0;
}
