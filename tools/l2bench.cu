// l2bench.cu — microbenchmark of random-access L2 operations on B200 (sm_100a):
// the scan's primitive is a 4-byte red.global.or into an L2-resident bitmap; this
// measures that primitive's ceiling (SURVEY §8(d) asks for a measured random-sector
// peak) and probes whether die-local addressing (L2 is split across the two dies)
// changes it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2bench tools/l2bench.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

template <int OP>
__global__ void k_random(uint32_t* buf, uint32_t nwords_log2, uint32_t iters, uint64_t seed) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint32_t mask = (1u << nwords_log2) - 1u;
  for (uint32_t it = 0; it < iters; ++it) {
    uint64_t h = mix(seed ^ (tid * 0x9E3779B97F4A7C15ULL) ^ ((uint64_t)it << 40));
    uint32_t w = (uint32_t)h & mask;
    uint32_t bit = 1u << ((h >> 32) & 31);
    if (OP == 0) atomicOr(buf + w, bit);
    else if (OP == 1) buf[w] = bit;
    else if (OP == 2) asm volatile("st.global.u8 [%0], %1;" :: "l"((uint8_t*)buf + ((h >> 8) & ((uint64_t)mask * 4 + 3))), "h"((uint16_t)1) : "memory");
    else atomicAdd(buf + w, 1u);
  }
}

// latency probe: one thread per block; measures the atomic latency to the first word
// of each chunk; records smid.
__global__ void k_probe(uint32_t* buf, uint32_t chunk_words, uint32_t n_chunks, uint32_t* lat,
                        uint32_t* smid_out) {
  if (threadIdx.x) return;
  uint32_t smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  smid_out[blockIdx.x] = smid;
  for (uint32_t c = 0; c < n_chunks; ++c) {
    // chain of 8 dependent atomics inside the chunk (the value returned, 0, feeds the
    // next address), timed as a whole
    uint32_t* base = buf + (size_t)c * chunk_words;
    uint32_t v = 0;
    long long t0 = clock64();
#pragma unroll
    for (int j = 0; j < 8; ++j) v = atomicAdd(base + 16 * j + v, 0u);
    long long t1 = clock64();
    if (v == 0xFFFFFFFF) buf[0] = v;
    lat[(size_t)blockIdx.x * n_chunks + c] = (uint32_t)((t1 - t0) / 8);
  }
}

// die-local variant: every SM only targets chunks in its die's list
__global__ void k_red_local(uint32_t* buf, const uint32_t* die_of_sm, const uint32_t* chunks0,
                            const uint32_t* chunks1, uint32_t n0, uint32_t n1, uint32_t chunk_words_log2,
                            uint32_t iters, uint64_t seed) {
  uint32_t smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  const uint32_t die = die_of_sm[smid];
  const uint32_t* lst = die ? chunks1 : chunks0;
  const uint32_t n = die ? n1 : n0;
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint32_t wmask = (1u << chunk_words_log2) - 1u;
  for (uint32_t it = 0; it < iters; ++it) {
    uint64_t h = mix(seed ^ (tid * 0x9E3779B97F4A7C15ULL) ^ ((uint64_t)it << 40));
    uint32_t c = lst[(uint32_t)(((h >> 32) * (uint64_t)n) >> 32)];
    uint32_t w = (c << chunk_words_log2) | ((uint32_t)h & wmask);
    atomicOr(buf + w, 1u << ((h >> 20) & 31));
  }
}

int main(int argc, char** argv) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const uint32_t iters = 256;
  const char* names[] = {"red.or.b32", "st.b32", "st.u8", "red.add.u32"};
  for (uint32_t lg : {20u, 22u, 24u, 25u, 26u}) {   // 4 MiB .. 256 MiB of words
    if (argc > 1) break;
    uint32_t* buf;
    CK(cudaMalloc(&buf, (size_t)4 << lg));
    CK(cudaMemset(buf, 0, (size_t)4 << lg));
    for (int op = 0; op < 4; ++op) {
      int blocks = sms * 8, threads = 256;
      for (int rep = 0; rep < 2; ++rep) {
        CK(cudaEventRecord(e0));
        if (op == 0) k_random<0><<<blocks, threads>>>(buf, lg, iters, rep);
        if (op == 1) k_random<1><<<blocks, threads>>>(buf, lg, iters, rep);
        if (op == 2) k_random<2><<<blocks, threads>>>(buf, lg, iters, rep);
        if (op == 3) k_random<3><<<blocks, threads>>>(buf, lg, iters, rep);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
        double ops = (double)blocks * threads * iters;
        if (rep == 1) printf("region %6.1f MiB  %-12s %7.1f Gop/s\n", (4.0 * (1u << lg)) / 1048576, names[op], ops / ms / 1e6);
      }
    }
    CK(cudaFree(buf));
  }
  // ---- die probe on a 16 MiB region with 2 KiB chunks
  const uint32_t chunk_words = 512, n_chunks = 8192;   // 16 MiB
  uint32_t* buf;
  CK(cudaMalloc(&buf, (size_t)chunk_words * n_chunks * 4));
  CK(cudaMemset(buf, 0, (size_t)chunk_words * n_chunks * 4));
  const int nb = sms * 2;
  uint32_t *lat, *smid;
  CK(cudaMalloc(&lat, (size_t)nb * n_chunks * 4));
  CK(cudaMalloc(&smid, nb * 4));
  k_probe<<<nb, 32>>>(buf, chunk_words, n_chunks, lat, smid);
  CK(cudaDeviceSynchronize());
  std::vector<uint32_t> hl((size_t)nb * n_chunks), hs(nb);
  CK(cudaMemcpy(hl.data(), lat, hl.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hs.data(), smid, nb * 4, cudaMemcpyDeviceToHost));
  // reference block 0: split chunks by its latency (threshold = midpoint of min/max clusters)
  std::vector<uint32_t> l0(hl.begin(), hl.begin() + n_chunks);
  std::vector<uint32_t> srt = l0;
  std::sort(srt.begin(), srt.end());
  printf("block0 smid %u latency pct: p5 %u p25 %u p50 %u p75 %u p95 %u\n", hs[0], srt[n_chunks / 20],
         srt[n_chunks / 4], srt[n_chunks / 2], srt[3 * n_chunks / 4], srt[19 * n_chunks / 20]);
  uint32_t thr = (srt[n_chunks / 4] + srt[3 * n_chunks / 4]) / 2;
  std::vector<int> near0(n_chunks);
  int cnt_near = 0;
  for (uint32_t c = 0; c < n_chunks; ++c) { near0[c] = l0[c] < thr; cnt_near += near0[c]; }
  printf("threshold %u: %d of %u chunks near block 0\n", thr, cnt_near, n_chunks);
  // classify every block (SM) by agreement with block 0's near set
  std::vector<uint32_t> die_of_sm(1024, 0);
  int agree_hist[11] = {0};
  for (int b = 0; b < nb; ++b) {
    int agree = 0;
    for (uint32_t c = 0; c < n_chunks; ++c) agree += ((hl[(size_t)b * n_chunks + c] < thr) == near0[c]);
    double f = (double)agree / n_chunks;
    agree_hist[(int)(f * 10)]++;
    die_of_sm[hs[b]] = f > 0.5 ? 0 : 1;
  }
  printf("agreement histogram (tenths):");
  for (int q = 0; q <= 10; ++q) printf(" %d", agree_hist[q]);
  printf("\n");
  std::vector<uint32_t> c0, c1;
  for (uint32_t c = 0; c < n_chunks; ++c) (near0[c] ? c0 : c1).push_back(c);
  uint32_t *d_die, *d_c0, *d_c1;
  CK(cudaMalloc(&d_die, 1024 * 4)); CK(cudaMalloc(&d_c0, c0.size() * 4 + 4)); CK(cudaMalloc(&d_c1, c1.size() * 4 + 4));
  CK(cudaMemcpy(d_die, die_of_sm.data(), 1024 * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_c0, c0.data(), c0.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_c1, c1.data(), c1.size() * 4, cudaMemcpyHostToDevice));
  for (int mode = 0; mode < 2; ++mode) {
    int blocks = sms * 8, threads = 256;
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaEventRecord(e0));
      if (mode == 0) k_random<0><<<blocks, threads>>>(buf, 22, iters, 7 + rep);
      else k_red_local<<<blocks, threads>>>(buf, d_die, d_c0, d_c1, (uint32_t)c0.size(), (uint32_t)c1.size(), 9, iters, 7 + rep);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
      if (rep) printf("16 MiB red.or %s: %.1f Gop/s\n", mode ? "die-local" : "uniform  ", (double)blocks * threads * iters / ms / 1e6);
    }
  }
  // same but with the opposite (far) assignment, as a control
  for (auto& d : die_of_sm) d ^= 1;
  CK(cudaMemcpy(d_die, die_of_sm.data(), 1024 * 4, cudaMemcpyHostToDevice));
  {
    int blocks = sms * 8, threads = 256;
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaEventRecord(e0));
      k_red_local<<<blocks, threads>>>(buf, d_die, d_c0, d_c1, (uint32_t)c0.size(), (uint32_t)c1.size(), 9, iters, 17 + rep);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
      if (rep) printf("16 MiB red.or die-far  : %.1f Gop/s\n", (double)blocks * threads * iters / ms / 1e6);
    }
  }
  return 0;
}
