// dsmembench.cu — throughput of random atomicOr into distributed shared memory (DSMEM)
// of a thread-block cluster, against local shared-memory atomics: decides whether a
// frame-partitioned scan whose cluster owns one frame's touch bitmap can beat k_scan_bin.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dsmembench tools/dsmembench.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

namespace cg = cooperative_groups;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// REMOTE = 0: atomics into the own CTA's shared memory; 1: into a random CTA of the cluster
template <int REMOTE>
__global__ void k_dsmem(uint32_t* out, uint32_t words_log2, uint32_t iters) {
  extern __shared__ uint32_t sm[];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t nwords = 1u << words_log2, mask = nwords - 1u;
  for (uint32_t q = threadIdx.x; q < nwords; q += blockDim.x) sm[q] = 0;
  cl.sync();
  const uint32_t csz = cl.num_blocks();
  uint32_t h = mix32((blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B9u + 7);
  for (uint32_t it = 0; it < iters; ++it) {
    h = mix32(h + it);
    uint32_t* base = sm;
    if (REMOTE) base = cl.map_shared_rank(sm, (h >> 24) % csz);
    atomicOr(base + (h & mask), 1u << (h >> 27));
  }
  cl.sync();
  uint32_t s = 0;
  for (uint32_t q = threadIdx.x; q < nwords; q += blockDim.x) s += sm[q];
  if (s == 0x12345678u) out[0] = s;
}

template <int REMOTE>
double run(int csz, int blocks, int threads, uint32_t wl2, uint32_t iters, uint32_t* out) {
  size_t smem = (size_t)4 << wl2;
  CK(cudaFuncSetAttribute(k_dsmem<REMOTE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (csz > 8) CK(cudaFuncSetAttribute(k_dsmem<REMOTE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csz; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  CK(cudaLaunchKernelEx(&cfg, k_dsmem<REMOTE>, out, wl2, iters));
  CK(cudaEventRecord(e0));
  CK(cudaLaunchKernelEx(&cfg, k_dsmem<REMOTE>, out, wl2, iters));
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  CK(cudaGetLastError());
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  return (double)blocks * threads * iters / ms / 1e6;
}

int main() {
  uint32_t* out;
  CK(cudaMalloc(&out, 64));
  for (int csz : {2, 4, 8, 16}) {
    for (uint32_t wl2 : {14u, 15u}) {
      int blocks = (144 / csz) * csz;
      double l = run<0>(csz, blocks, 512, wl2, 2048, out);
      double r = run<1>(csz, blocks, 512, wl2, 2048, out);
      printf("cluster %2d  smem %3u KiB  blocks %d: local atomicOr %8.1f G/s   DSMEM random-rank atomicOr %8.1f G/s\n",
             csz, (4u << wl2) >> 10, blocks, l, r);
    }
  }
  return 0;
}
