/*
 * asse_gen.h — seeded, counter-based synthetic packet-pair generator.
 *
 * This module is INPUT INFRASTRUCTURE shared by the CPU oracle side (tests,
 * bench cpu_baseline) and the GPU side (bench inputs). It holds none of the
 * ASSE method's arithmetic: no mangling, no BH, no AT codes. Every packet is a
 * pure function of (descriptor, slice t, slot j), so host and device produce
 * bit-identical streams and any shard/sample can be regenerated on its own.
 *
 * The CAIDA / CERNET traces the paper measures on (PAPER.md P:433, P:486,
 * P:162) are not available; the presets below stand in for them with the
 * shapes BASELINE.json.configs names (SURVEY.md §8(d) G1–G7). The recipe is
 * restated in DESIGN.md §3.
 *
 * Mixer choice: murmur3's fmix64 (not SplitMix64's finalizer, which both
 * method sides use for BH) so the generator's randomness is never correlated
 * with the sketch's hash functions.
 */
#ifndef ASSE_GEN_H
#define ASSE_GEN_H
#include <stdint.h>

#ifdef __CUDACC__
#define GEN_HD __host__ __device__ __forceinline__
#else
#define GEN_HD static inline
#endif

/* Generator kinds (BASELINE.json.configs[0..4]) */
enum {
  GEN_KIND_ZIPF_PLANTED = 1, /* C1: Zipf pool + planted hosts, fixed per-slice fresh bips */
  GEN_KIND_ZIPF_LOGU = 2,    /* C2: Zipf pool + planted hosts with log-uniform window card. */
  GEN_KIND_BACKBONE = 3,     /* C3/C5: Pareto peer sets, scanners, duplicates */
  GEN_KIND_DDOS = 4          /* C4: C3 mixture + bursting DDoS victims */
};

/* Stream tags (G1) */
enum {
  GT_HOSTID = 1, GT_BG = 2, GT_BIP = 3, GT_PERM = 4, GT_FRESH = 5, GT_CLASS = 6,
  GT_PEERIDX = 7, GT_PEER = 8, GT_SCAN = 9, GT_SCANBIP = 10, GT_DUP = 11, GT_NA = 12,
  GT_PLANT = 13, GT_VICTIM = 14
};

/* Plain-old-data descriptor; pointers are host or device copies of the tables. */
typedef struct {
  int32_t kind;
  uint32_t T;               /* slices in the run */
  uint64_t seed;
  uint64_t N;               /* packets per slice (whole job) */
  uint32_t k;               /* window length (C2 planted per-slice share n_p/k) */
  uint32_t n_hosts;         /* Zipf pool size (C1/C2) or background aip count (C3-C5) */
  const uint64_t* cdf;      /* n_hosts inclusive thresholds: pick smallest a with u < cdf[a] */
  const uint32_t* n_a;      /* C3-C5: per-aip peer-set size (G4) */
  uint32_t n_planted;       /* C1: 4, C2: 200 */
  const uint64_t* plant_off;/* n_planted+1 prefix sums of per-slice planted packets */
  uint64_t plant_total;     /* plant_off[n_planted] */
  uint32_t plant_stride;    /* fresh-bip counter stride per (t, host) */
  uint32_t n_scanners;      /* C3-C5: 50 */
  uint32_t pct_bg, pct_scan;/* class split in 1/2^24 units: bg < pct_bg, scan < pct_bg+pct_scan */
  uint32_t n_victims;       /* C4: 20 */
  uint32_t victim_pkts;     /* C4: 1000 per victim per active slice */
  uint32_t victim_span;     /* C4: 50 slices */
  const uint32_t* victim_on;/* C4: per-victim onset slice */
  uint32_t perm_bits;       /* even bit width of the cycle-walking slot permutation domain */
  uint32_t pad;
} gen_desc;

/* G1: 64-bit counter hash */
GEN_HD uint64_t gen_fmix64(uint64_t k) {
  k ^= k >> 33; k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33; return k;
}
GEN_HD uint64_t gen_key(uint64_t seed, uint64_t tag, uint64_t t) {
  return gen_fmix64(gen_fmix64(seed ^ (tag * 0xD6E8FEB86659FD93ULL)) ^ (t * 0xA0761D6478BD642FULL));
}
/* distinct j -> distinct outputs for a fixed key (j*odd and fmix64 are bijections) */
GEN_HD uint64_t gen_h(uint64_t key, uint64_t j) {
  return gen_fmix64(key ^ (j * 0x9E3779B97F4A7C15ULL));
}

/* G2: keyed bijection on b-bit values (b even, 2..32), 4-round balanced Feistel. */
GEN_HD uint32_t gen_feistel(uint64_t key, uint32_t x, uint32_t bits) {
  const uint32_t hb = bits >> 1;
  const uint32_t m = (hb >= 32) ? 0xFFFFFFFFu : ((1u << hb) - 1u);
  uint32_t L = (x >> hb) & m, R = x & m;
  for (uint32_t rd = 0; rd < 4; ++rd) {
    uint32_t f = (uint32_t)(gen_fmix64(key ^ (((uint64_t)rd << 40) | R)) >> 17) & m;
    uint32_t nl = R;
    R = L ^ f;
    L = nl;
  }
  return (uint32_t)(((uint64_t)L << hb) | R);
}
/* host id: distinct u32 for distinct index (never an affine map; G2) */
GEN_HD uint32_t gen_host_id(uint64_t seed, uint32_t idx) {
  return gen_feistel(gen_key(seed, GT_HOSTID, 0), idx, 32);
}
/* fresh bip: distinct u32 for distinct counter value */
GEN_HD uint32_t gen_fresh_bip(uint64_t seed, uint32_t ctr) {
  return gen_feistel(gen_key(seed, GT_FRESH, 0), ctr, 32);
}
/* Cycle-walking permutation of [0, n) inside a perm_bits domain (n <= 2^perm_bits). */
GEN_HD uint64_t gen_perm(uint64_t key, uint64_t j, uint64_t n, uint32_t bits) {
  uint32_t x = (uint32_t)j;
  do { x = gen_feistel(key, x, bits); } while ((uint64_t)x >= n);
  return x;
}
/* G3: smallest a with u < cdf[a]; clamps to n-1 */
GEN_HD uint32_t gen_cdf_search(const uint64_t* cdf, uint32_t n, uint64_t u) {
  uint32_t lo = 0, hi = n - 1;
  while (lo < hi) {
    uint32_t mid = lo + ((hi - lo) >> 1);
    if (u < cdf[mid]) hi = mid; else lo = mid + 1;
  }
  return lo;
}
/* multiply-shift reduction of a 32-bit uniform to [0, n) */
GEN_HD uint32_t gen_reduce(uint32_t h32, uint32_t n) {
  return (uint32_t)(((uint64_t)h32 * (uint64_t)n) >> 32);
}

/* C3 mixture slot (no duplicate class): background or scanner. */
GEN_HD void gen_backbone_fresh(const gen_desc* d, uint32_t t, uint64_t j, uint32_t cls_u,
                               uint32_t* aip, uint32_t* bip) {
  if (cls_u < d->pct_bg) {
    uint64_t ua = gen_h(gen_key(d->seed, GT_BG, t), j);
    uint32_t a = gen_cdf_search(d->cdf, d->n_hosts, ua);
    uint32_t id = gen_host_id(d->seed, a);
    uint32_t na = d->n_a[a];
    uint32_t jj = gen_reduce((uint32_t)(gen_h(gen_key(d->seed, GT_PEERIDX, t), j) >> 32), na);
    /* G5: peer set of aip a is fixed across slices */
    *aip = id;
    *bip = (uint32_t)gen_h(gen_key(d->seed, GT_PEER, a), jj);
  } else {
    uint64_t hs = gen_h(gen_key(d->seed, GT_SCAN, t), j);
    uint32_t s = gen_reduce((uint32_t)(hs >> 32), d->n_scanners);
    *aip = gen_host_id(d->seed, d->n_hosts + s);
    *bip = (uint32_t)gen_h(gen_key(d->seed, GT_SCANBIP, t), j);
  }
}
GEN_HD uint32_t gen_class_u(const gen_desc* d, uint32_t t, uint64_t j) {
  return (uint32_t)(gen_h(gen_key(d->seed, GT_CLASS, t), j) >> 40); /* 24-bit uniform */
}
/* C3: background 75% / scanners 5% / duplicates 20% (G6, G7) */
GEN_HD void gen_backbone(const gen_desc* d, uint32_t t, uint64_t j, uint32_t* aip, uint32_t* bip) {
  uint32_t cu = gen_class_u(d, t, j);
  if (cu >= d->pct_bg + d->pct_scan) {
    /* duplicate: copy a uniformly chosen non-duplicate slot of the same slice */
    uint64_t kd = gen_key(d->seed, GT_DUP, t);
    uint64_t jp = j;
    uint32_t cp = cu;
    for (uint32_t att = 0; att < 64; ++att) {
      uint64_t h = gen_h(kd, j * 64 + att);
      jp = (uint64_t)(((unsigned __int128)h * d->N) >> 64);
      cp = gen_class_u(d, t, jp);
      if (cp < d->pct_bg + d->pct_scan) break;
    }
    if (cp >= d->pct_bg + d->pct_scan) cp = 0; /* astronomically rare: treat as background */
    gen_backbone_fresh(d, t, jp, cp, aip, bip);
    return;
  }
  gen_backbone_fresh(d, t, j, cu, aip, bip);
}

/* One packet (aip, bip) of slice t, slot j in [0, N). */
GEN_HD void gen_packet(const gen_desc* d, uint32_t t, uint64_t j, uint32_t* aip, uint32_t* bip) {
  if (d->kind == GEN_KIND_ZIPF_PLANTED || d->kind == GEN_KIND_ZIPF_LOGU) {
    uint64_t p = gen_perm(gen_key(d->seed, GT_PERM, t), j, d->N, d->perm_bits);
    if (p < d->plant_total) {
      /* planted packet p -> (host h, message m) via prefix sums */
      uint32_t lo = 0, hi = d->n_planted - 1;
      while (lo < hi) {
        uint32_t mid = (lo + hi + 1) >> 1;
        if (d->plant_off[mid] <= p) lo = mid; else hi = mid - 1;
      }
      uint32_t m = (uint32_t)(p - d->plant_off[lo]);
      *aip = gen_host_id(d->seed, d->n_hosts + lo);
      *bip = gen_fresh_bip(d->seed, (t * d->n_planted + lo) * d->plant_stride + m);
      return;
    }
    uint64_t ub = gen_h(gen_key(d->seed, GT_BG, t), p);
    uint32_t r = gen_cdf_search(d->cdf, d->n_hosts, ub);
    *aip = gen_host_id(d->seed, r);
    *bip = (uint32_t)gen_h(gen_key(d->seed, GT_BIP, t), p);
    return;
  }
  if (d->kind == GEN_KIND_DDOS) {
    uint64_t p = gen_perm(gen_key(d->seed, GT_PERM, t), j, d->N, d->perm_bits);
    uint64_t nv = (uint64_t)d->n_victims * d->victim_pkts;
    if (p < nv) {
      uint32_t v = (uint32_t)(p / d->victim_pkts), m = (uint32_t)(p % d->victim_pkts);
      uint32_t on = d->victim_on[v];
      if (t >= on && t < on + d->victim_span) {
        *aip = gen_host_id(d->seed, d->n_hosts + d->n_scanners + v);
        *bip = gen_fresh_bip(d->seed, (t * d->n_victims + v) * d->victim_pkts + m);
        return;
      }
    }
    gen_backbone(d, t, j, aip, bip);
    return;
  }
  gen_backbone(d, t, j, aip, bip);
}

#endif /* ASSE_GEN_H */
