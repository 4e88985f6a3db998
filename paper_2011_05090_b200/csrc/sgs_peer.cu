// Peer-memory exchange of a row-sharded state (one node, NVLink / NVSwitch):
// allocation of the exchange area, CUDA IPC export / import, the device
// descriptor the LS kernel reads, and the generation bump that opens a
// factorisation.  The exchange itself runs inside ls_step_kernel (sgs_rgs.cu).

#include <cstring>

#include "sgs_common.cuh"

namespace sgs {

__global__ void peer_begin_kernel(const sgs_peer_desc_dev* d) {
  // own area: bump the flag generation (every rank does the same, in step)
  unsigned int* gen = reinterpret_cast<unsigned int*>(d->area[d->rank]);
  *gen = *gen + 1u;
}

}  // namespace sgs

using namespace sgs;

extern "C" int64_t sgs_peer_bytes(int world, int k, int cl) {
  if (world < 1 || world > kPeerMaxWorld || k < 1 || cl < 1 || cl > kPeerMaxCl) return 0;
  return peer_area_bytes(world, k);
}

extern "C" int sgs_peer_alloc(int64_t bytes, void** area) {
  SGS_REQUIRE(area && bytes > 0, "peer_alloc: bad args");
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, (size_t)bytes);  // its own allocation: IPC-exportable
  if (e == cudaSuccess) e = cudaMemset(p, 0, (size_t)bytes);
  if (e != cudaSuccess) {
    set_error("peer_alloc: %s", cudaGetErrorString(e));
    cudaGetLastError();
    return SGS_ECUDA;
  }
  *area = p;
  return 0;
}

extern "C" int sgs_peer_free(void* area) {
  SGS_REQUIRE(area, "peer_free: null");
  return check_ex(cudaFree(area), "peer_free");
}

extern "C" int sgs_peer_export(void* area, unsigned char* handle64) {
  SGS_REQUIRE(area && handle64, "peer_export: null");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, area);
  if (e != cudaSuccess) return check_ex(e, "peer_export");
  memcpy(handle64, &h, 64);
  return 0;
}

extern "C" int sgs_peer_import(const unsigned char* handle64, void** area) {
  SGS_REQUIRE(area && handle64, "peer_import: null");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  const cudaError_t e = cudaIpcOpenMemHandle(area, h, cudaIpcMemLazyEnablePeerAccess);
  return check_ex(e, "peer_import");
}

extern "C" int sgs_peer_unimport(void* area) {
  SGS_REQUIRE(area, "peer_unimport: null");
  return check_ex(cudaIpcCloseMemHandle(area), "peer_unimport");
}

extern "C" int sgs_peer_desc_create(int world, int rank, int k, void* const* areas, void** desc) {
  SGS_REQUIRE(world >= 1 && world <= kPeerMaxWorld && rank >= 0 && rank < world && k >= 1 &&
                  areas && desc,
              "peer_desc_create: bad args (world <= %d)", kPeerMaxWorld);
  sgs_peer_desc_dev h{};
  h.world = world;
  h.rank = rank;
  h.k = k;
  for (int q = 0; q < world; ++q) {
    SGS_REQUIRE(areas[q] != nullptr, "peer_desc_create: area %d missing", q);
    h.area[q] = static_cast<unsigned char*>(areas[q]);
  }
  void* d = nullptr;
  cudaError_t e = cudaMalloc(&d, sizeof(h));
  if (e == cudaSuccess) e = cudaMemcpy(d, &h, sizeof(h), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return check_ex(e, "peer_desc_create");
  *desc = d;
  return 0;
}

extern "C" int sgs_peer_desc_free(void* desc) {
  SGS_REQUIRE(desc, "peer_desc_free: null");
  return check_ex(cudaFree(desc), "peer_desc_free");
}

extern "C" int sgs_peer_begin(void* desc, void* stream) {
  SGS_REQUIRE(desc, "peer_begin: null");
  peer_begin_kernel<<<1, 1, 0, as_stream(stream)>>>(static_cast<const sgs_peer_desc_dev*>(desc));
  return check_launch("peer_begin_kernel");
}
