// smembench.cu — per-SM throughput of the primitives a binned scan would be built from
// (shared-memory atomics, random shared stores/loads, warp match, coalesced global
// stores into an L2-resident ring), next to the random red.global.or the scan uses now.
// It decides whether binning updates before they reach L2 can beat one RED per update.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/smembench tools/smembench.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// OP 0: atomicOr smem word; 1: st.shared.u8; 2: st.shared.b32; 3: ld.shared.b32 (sum);
// 4: racy ld/or/st; 5: match.any on a 10-bit key; 6: red.global.or (16 MiB region)
template <int OP>
__global__ void k_smem(uint32_t* out, uint32_t* gbuf, uint32_t words_log2, uint32_t iters, uint32_t seed) {
  extern __shared__ uint32_t sm[];
  const uint32_t nwords = 1u << words_log2, mask = nwords - 1u;
  for (uint32_t q = threadIdx.x; q < nwords; q += blockDim.x) sm[q] = 0;
  __syncthreads();
  uint32_t acc = 0;
  uint32_t h = mix32(seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B9u);
#pragma unroll 4
  for (uint32_t it = 0; it < iters; ++it) {
    h = mix32(h + it);
    const uint32_t w = h & mask;
    if (OP == 0) atomicOr(sm + w, 1u << (h >> 27));
    else if (OP == 1) reinterpret_cast<volatile uint8_t*>(sm)[(h >> 3) & (mask * 4 + 3)] = 1;
    else if (OP == 2) reinterpret_cast<volatile uint32_t*>(sm)[w] = h;
    else if (OP == 3) acc += reinterpret_cast<volatile uint32_t*>(sm)[w];
    else if (OP == 4) { volatile uint32_t* v = sm; v[w] = v[w] | (1u << (h >> 27)); }
    else if (OP == 5) acc += __match_any_sync(0xffffffffu, h >> 22);
    else atomicOr(gbuf + (h & ((1u << 22) - 1u)), 1u << (h >> 27));
  }
  __syncthreads();
  uint32_t s = acc;
  for (uint32_t q = threadIdx.x; q < nwords; q += blockDim.x) s += sm[q];
  if (s == 0x12345678u) out[0] = s;
}

// coalesced 16-B stores / loads streaming through a ring of ring_bytes (L2-resident if small)
__global__ void k_stv4(uint4* ring, uint64_t ring_v4, uint32_t iters) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  for (uint32_t it = 0; it < iters; ++it) {
    uint64_t idx = (tid + it * nth) % ring_v4;
    ring[idx] = make_uint4(it, (uint32_t)tid, 1, 2);
  }
}
__global__ void k_ldv4(const uint4* ring, uint64_t ring_v4, uint32_t iters, uint32_t* out) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (uint32_t it = 0; it < iters; ++it) {
    uint64_t idx = (tid + it * nth) % ring_v4;
    uint4 v = ring[idx];
    acc += v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int OP>
double run_smem(int blocks, int threads, uint32_t wl2, uint32_t iters, uint32_t* out, uint32_t* gbuf) {
  size_t smem = (size_t)4 << wl2;
  CK(cudaFuncSetAttribute(k_smem<OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  k_smem<OP><<<blocks, threads, smem>>>(out, gbuf, wl2, iters, 1);
  CK(cudaEventRecord(e0));
  k_smem<OP><<<blocks, threads, smem>>>(out, gbuf, wl2, iters, 2);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  CK(cudaGetLastError());
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  return (double)blocks * threads * iters / ms / 1e6;   // G lane-ops/s
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint32_t *out, *gbuf;
  CK(cudaMalloc(&out, 64));
  CK(cudaMalloc(&gbuf, 16u << 20));
  CK(cudaMemset(gbuf, 0, 16u << 20));
  const char* names[] = {"atom.shared.or (ATOMS)", "st.shared.u8", "st.shared.b32", "ld.shared.b32",
                         "ld/or/st.shared (racy)", "match.any.sync", "red.global.or 16MiB"};
  for (uint32_t wl2 : {14u, 15u}) {       // 64 KiB / 128 KiB of shared memory per CTA
    for (int occ : {1, 2}) {
      if (wl2 == 15 && occ == 2) continue;
      int threads = 1024 / occ > 512 ? 512 : 1024 / occ;
      int blocks = sms * occ;
      uint32_t iters = 4096;
      double r[7];
      r[0] = run_smem<0>(blocks, threads, wl2, iters, out, gbuf);
      r[1] = run_smem<1>(blocks, threads, wl2, iters, out, gbuf);
      r[2] = run_smem<2>(blocks, threads, wl2, iters, out, gbuf);
      r[3] = run_smem<3>(blocks, threads, wl2, iters, out, gbuf);
      r[4] = run_smem<4>(blocks, threads, wl2, iters, out, gbuf);
      r[5] = run_smem<5>(blocks, threads, wl2, iters, out, gbuf);
      r[6] = run_smem<6>(blocks, threads, wl2, iters / 8, out, gbuf);
      for (int o = 0; o < 7; ++o)
        printf("smem %3u KiB/CTA occ %d threads %d  %-26s %8.1f G lane-op/s  (%.2f SM-cyc/lane @1965MHz)\n",
               (4u << wl2) >> 10, occ, threads, names[o], r[o], sms * 1.965 / r[o]);
    }
  }
  // coalesced streaming into a ring
  for (uint64_t ring_mb : {32ull, 64ull, 1024ull}) {
    uint4* ring;
    CK(cudaMalloc(&ring, ring_mb << 20));
    uint64_t nv4 = (ring_mb << 20) / 16;
    int blocks = sms * 4, threads = 512;
    uint32_t iters = (uint32_t)((4ull << 30) / 16 / ((uint64_t)blocks * threads));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    for (int op = 0; op < 2; ++op) {
      for (int rep = 0; rep < 2; ++rep) {
        CK(cudaEventRecord(e0));
        if (op == 0) k_stv4<<<blocks, threads>>>(ring, nv4, iters);
        else k_ldv4<<<blocks, threads>>>(ring, nv4, iters, out);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
        if (rep) printf("ring %5llu MiB  %s v4 coalesced: %8.1f GB/s\n", (unsigned long long)ring_mb,
                        op ? "ld" : "st", (double)blocks * threads * iters * 16 / ms / 1e6);
      }
    }
    CK(cudaFree(ring));
  }
  return 0;
}
