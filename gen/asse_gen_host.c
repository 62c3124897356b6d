/*
 * asse_gen_host.c — host half of the synthetic trace generator (input
 * infrastructure; holds none of ASSE's arithmetic). Builds the per-preset
 * sampling tables once and fills packet buffers as a pure function of
 * (preset, seed, slice, slot). Presets follow BASELINE.json.configs[0..4] and
 * SURVEY.md §8(d); DESIGN.md §3 restates the recipe.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include "gen_internal.h"

static uint32_t even_bits_for(uint64_t n) {
  uint32_t b = 2;
  while (b < 32 && ((uint64_t)1 << b) < n) b += 2;
  return b;
}

/* G3: Zipf(s) over n ranks; cdf[r] = floor(2^64 * P(rank <= r)), last = 2^64-1 */
static void build_zipf(uint64_t* cdf, uint32_t n, double s) {
  long double S = 0.0L;
  for (uint32_t r = 0; r < n; ++r) S += 1.0L / powl((long double)(r + 1), (long double)s);
  long double acc = 0.0L;
  const long double two64 = 18446744073709551616.0L;
  for (uint32_t r = 0; r < n; ++r) {
    acc += 1.0L / powl((long double)(r + 1), (long double)s);
    long double v = acc / S * two64;
    cdf[r] = (v >= two64) ? UINT64_MAX : (uint64_t)v;
  }
  cdf[n - 1] = UINT64_MAX;
}

/* G4: Pareto(alpha, x_m=1) peer-set sizes, capped at 2^20; aip chosen prop. to n_a */
static void build_backbone(gen_ctx* g, uint64_t seed, uint32_t n, double alpha) {
  g->n_a = (uint32_t*)malloc(sizeof(uint32_t) * n);
  g->cdf = (uint64_t*)malloc(sizeof(uint64_t) * n);
  g->n_a_n = n;
  g->cdf_n = n;
  uint64_t key = gen_key(seed, GT_NA, 0);
  unsigned __int128 total = 0;
  for (uint32_t a = 0; a < n; ++a) {
    uint64_t h = gen_h(key, a);
    double U = (double)((h >> 11) + 1) / 9007199254740992.0; /* (0, 1] */
    double x = floor(pow(U, -1.0 / alpha));
    uint32_t na = (x >= 1048576.0) ? 1048576u : (uint32_t)x;
    if (na < 1) na = 1;
    g->n_a[a] = na;
    total += na;
  }
  unsigned __int128 acc = 0;
  for (uint32_t a = 0; a < n; ++a) {
    acc += g->n_a[a];
    unsigned __int128 v = (acc << 64) / total;
    g->cdf[a] = (v >> 64) ? UINT64_MAX : (uint64_t)v;
  }
  g->cdf[n - 1] = UINT64_MAX;
}

gen_ctx* gen_new(int preset, uint64_t seed, uint64_t N, uint32_t T) {
  gen_ctx* g = (gen_ctx*)calloc(1, sizeof(gen_ctx));
  gen_desc* d = &g->host;
  g->preset = preset;
  d->seed = seed;
  switch (preset) {
    case 1: { /* C1: k=4, 8x200k, Zipf(1.1) over 16384, 4 planted x 600 fresh bips per slice */
      d->kind = GEN_KIND_ZIPF_PLANTED;
      d->N = N ? N : 200000; d->T = T ? T : 8; d->k = 4;
      d->n_hosts = 16384;
      g->cdf = (uint64_t*)malloc(sizeof(uint64_t) * d->n_hosts); g->cdf_n = d->n_hosts;
      build_zipf(g->cdf, d->n_hosts, 1.1);
      d->n_planted = 4; d->plant_stride = 600;
      g->plant_off = (uint64_t*)malloc(sizeof(uint64_t) * 5); g->plant_n = 5;
      for (int h = 0; h <= 4; ++h) g->plant_off[h] = (uint64_t)h * 600;
      break;
    }
    case 2: { /* C2: k=10, 30x2M, Zipf(1.2) over 1M, 200 planted n_p ~ logU[512,65536] */
      d->kind = GEN_KIND_ZIPF_LOGU;
      d->N = N ? N : 2000000; d->T = T ? T : 30; d->k = 10;
      d->n_hosts = 1000000;
      g->cdf = (uint64_t*)malloc(sizeof(uint64_t) * d->n_hosts); g->cdf_n = d->n_hosts;
      build_zipf(g->cdf, d->n_hosts, 1.2);
      d->n_planted = 200; d->plant_stride = 8192;
      g->plant_off = (uint64_t*)malloc(sizeof(uint64_t) * 201); g->plant_n = 201;
      uint64_t kp = gen_key(seed, GT_PLANT, 0);
      g->plant_off[0] = 0;
      for (uint32_t h = 0; h < 200; ++h) {
        double U = (double)(gen_h(kp, h) >> 11) / 9007199254740992.0; /* [0,1) */
        double np = exp(log(512.0) + U * (log(65536.0) - log(512.0)));
        uint32_t m = (uint32_t)llround(np / (double)d->k);
        if (m < 1) m = 1;
        g->plant_off[h + 1] = g->plant_off[h] + m;
      }
      break;
    }
    case 3: case 5: { /* C3 (k=60, 300x20M) / C5 (120x100M): 4M Pareto aips, scanners, dups */
      d->kind = GEN_KIND_BACKBONE;
      d->N = N ? N : (preset == 3 ? 20000000ull : 100000000ull);
      d->T = T ? T : (preset == 3 ? 300 : 120);
      d->k = 60;
      d->n_hosts = 4000000;
      build_backbone(g, seed, d->n_hosts, 1.3);
      d->n_scanners = 50;
      break;
    }
    case 4: { /* C4: k=300, 600x10M, C3 mixture + 20 DDoS victims x 50-slice spans */
      d->kind = GEN_KIND_DDOS;
      d->N = N ? N : 10000000ull; d->T = T ? T : 600; d->k = 300;
      d->n_hosts = 4000000;
      build_backbone(g, seed, d->n_hosts, 1.3);
      d->n_scanners = 50;
      d->n_victims = 20; d->victim_pkts = 1000; d->victim_span = 50;
      g->victim_on = (uint32_t*)malloc(sizeof(uint32_t) * 20); g->victim_n = 20;
      uint64_t kv = gen_key(seed, GT_VICTIM, 0);
      for (uint32_t v = 0; v < 20; ++v)
        g->victim_on[v] = gen_reduce((uint32_t)(gen_h(kv, v) >> 32), 250);
      break;
    }
    default:
      free(g);
      return NULL;
  }
  d->pct_bg = 12582912u;  /* 0.75 * 2^24 */
  d->pct_scan = 838861u;  /* 0.05 * 2^24 */
  d->cdf = g->cdf;
  d->n_a = g->n_a;
  d->plant_off = g->plant_off;
  d->plant_total = g->plant_off ? g->plant_off[d->n_planted] : 0;
  d->victim_on = g->victim_on;
  d->perm_bits = even_bits_for(d->N);
  return g;
}

void gen_free(gen_ctx* g);  /* defined in the CUDA twin (frees device copies too) */

const gen_desc* gen_host_desc(const gen_ctx* g) { return &g->host; }
uint64_t gen_get_N(const gen_ctx* g) { return g->host.N; }
uint32_t gen_get_T(const gen_ctx* g) { return g->host.T; }
uint32_t gen_get_k(const gen_ctx* g) { return g->host.k; }
uint32_t gen_get_n_a(const gen_ctx* g, uint32_t a) { return g->n_a ? g->n_a[a] : 0; }
uint64_t gen_plant_total(const gen_ctx* g) { return g->host.plant_total; }
uint32_t gen_planted_id(const gen_ctx* g, uint32_t h) {
  return gen_host_id(g->host.seed, g->host.n_hosts + h);
}
uint32_t gen_planted_m(const gen_ctx* g, uint32_t h) {
  return (uint32_t)(g->plant_off[h + 1] - g->plant_off[h]);
}
uint32_t gen_victim_id(const gen_ctx* g, uint32_t v) {
  return gen_host_id(g->host.seed, g->host.n_hosts + g->host.n_scanners + v);
}
uint32_t gen_victim_onset(const gen_ctx* g, uint32_t v) { return g->victim_on[v]; }
uint32_t gen_scanner_id(const gen_ctx* g, uint32_t s) {
  return gen_host_id(g->host.seed, g->host.n_hosts + s);
}
uint32_t gen_pool_id(const gen_ctx* g, uint32_t idx) { return gen_host_id(g->host.seed, idx); }

/* Fill out[2m], out[2m+1] = packet of slot j0 + m*stride of slice t, m in [0, n). */
void gen_fill(const gen_ctx* g, uint32_t t, uint64_t j0, uint64_t stride, uint64_t n,
              uint32_t* out, int nthreads) {
  const gen_desc* d = &g->host;
#ifdef _OPENMP
  if (nthreads > 0) {
#pragma omp parallel for schedule(static) num_threads(nthreads)
    for (long long m = 0; m < (long long)n; ++m)
      gen_packet(d, t, j0 + (uint64_t)m * stride, &out[2 * m], &out[2 * m + 1]);
    return;
  }
#endif
  for (uint64_t m = 0; m < n; ++m) gen_packet(d, t, j0 + m * stride, &out[2 * m], &out[2 * m + 1]);
}
