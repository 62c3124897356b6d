/*
 * asse_gen_cuda.cu — device twin of the synthetic trace generator (input
 * infrastructure only). The same gen_packet() from asse_gen.h runs here, so
 * the device stream is bit-identical to gen_fill() on the host; tests check
 * that on samples. Used by bench.py / tests to create device-resident slices.
 */
#include <cuda_runtime.h>
#include <stdlib.h>
#include "gen_internal.h"

extern "C" {

static int up(void** dst, const void* src, size_t bytes) {
  if (!src || !bytes) { *dst = nullptr; return 0; }
  if (cudaMalloc(dst, bytes) != cudaSuccess) return -1;
  if (cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess) return -1;
  return 0;
}

int gen_cuda_upload(gen_ctx* g) {
  if (g->uploaded) return 0;
  if (up(&g->d_cdf, g->cdf, g->cdf_n * 8) || up(&g->d_n_a, g->n_a, g->n_a_n * 4) ||
      up(&g->d_plant_off, g->plant_off, g->plant_n * 8) ||
      up(&g->d_victim_on, g->victim_on, g->victim_n * 4))
    return -1;
  g->dev = g->host;
  g->dev.cdf = (const uint64_t*)g->d_cdf;
  g->dev.n_a = (const uint32_t*)g->d_n_a;
  g->dev.plant_off = (const uint64_t*)g->d_plant_off;
  g->dev.victim_on = (const uint32_t*)g->d_victim_on;
  g->uploaded = 1;
  return 0;
}

void gen_free(gen_ctx* g) {
  if (!g) return;
  if (g->uploaded) {
    cudaFree(g->d_cdf); cudaFree(g->d_n_a); cudaFree(g->d_plant_off); cudaFree(g->d_victim_on);
  }
  free(g->cdf); free(g->n_a); free(g->plant_off); free(g->victim_on);
  free(g);
}

}  // extern "C"

__global__ void k_gen_fill(gen_desc d, uint32_t t, uint64_t j0, uint64_t stride, uint64_t n,
                           uint2* __restrict__ out) {
  for (uint64_t m = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; m < n;
       m += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t a, b;
    gen_packet(&d, t, j0 + m * stride, &a, &b);
    out[m] = make_uint2(a, b);
  }
}

extern "C" int gen_cuda_fill(gen_ctx* g, uint32_t t, uint64_t j0, uint64_t stride, uint64_t n,
                             uint32_t* d_out, void* stream) {
  if (gen_cuda_upload(g)) return -1;
  if (n == 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t blocks = (n + 255) / 256;
  if (blocks > (uint64_t)sms * 16) blocks = (uint64_t)sms * 16;
  k_gen_fill<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(g->dev, t, j0, stride, n,
                                                                   (uint2*)d_out);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
