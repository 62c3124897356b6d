/*
 * asse_oracle.c — plain, slow, single-threaded CPU oracle of ASSE's hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this. It shares no
 * code, header, table or constant generator with the CUDA path
 * (paper_1807_01527_b200/csrc); neither side includes the other.
 *
 * It follows "Distributed super point cardinality estimation under sliding
 * time window for high speed network" (PAPER.md = /root/reference/PAPER.md,
 * cited as P:<line>) step by step, in the paper's order and notation, in the
 * readings listed in SURVEY.md §8(c) (A1..A35) and DESIGN.md §2:
 *
 *   step 0  init     InitAT; ATV blocks a,b and ACT (A7)
 *   step 1  scan     Alg. 3 "Scan IP pair", RRH
 *   step 2  weights  Alg. 1 checkAT; |ATV|^{k'}; AAT
 *   step 3  SA       super ATV: w >= g - g e^{-theta/g}
 *   step 4  restore  Alg. 4, duplicate-bit check done as soon as
 *                    two rows are assigned (same set; A16)
 *   step 5  estimate Alg. 5 NAT; Eq. 4 UP; Eq. 5
 *   step 6  report   ascending ip (A24); mode 0 keeps est >= theta (A21)
 *   step 7  advance  ACT+1, Alg. 2 preserveAT
 *
 * Floating point is double (A25). Parity pins are in tests/test_oracle_*.py.
 * Every function here has a pin except where its header says "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_E_PARAM (-1)
#define ORACLE_E_CAPACITY (-3)
#define ORACLE_E_OVERFLOW (-4)

typedef struct {
  uint32_t k, k_prime, r, c, u, s, g;
  double theta;
  uint64_t seed;
  uint32_t max_candidates;
  uint32_t mangle;       /* 0: f(x) = A x mod 2^32, A odd (A8); 1: f(x) = A x mod p,
                            p = 2^32 + 15 prime, cycle-walked into 32 bits (P:305 literal) */
} oracle_params;

typedef struct {
  uint32_t ip, nat;
  double estimate;
  uint32_t flags, pad;
} oracle_report; /* flags: 1 = SATURATED (nat == g), 2 = ABOVE_THETA (estimate >= theta) */

typedef struct {
  oracle_params p;
  uint32_t F, E;          /* frames 2^u, columns 2^c */
  uint32_t a, b;          /* ATV block sizes */
  uint32_t C0;            /* ACT of block 0 */
  uint64_t t;             /* current slice */
  uint64_t A, A_inv;      /* mangling key and inverse (A8 or mod p) */
  uint64_t K_bh;          /* BH key (A13) */
  uint16_t* pool;         /* AT[y][z][x][i] */
  /* per-slice end results */
  uint32_t* w;            /* |ATV|^{k'} per [y][z][x] */
  uint64_t* aat;          /* |AAT(k',y,z)| */
  uint8_t* super;         /* super flag per [y][z][x] */
  oracle_report* rep;     /* CSIP reports of the last end_slice, ascending ip */
  uint32_t n_rep, cap_rep;
} oracle_t;

/* ------------------------------------------------------------------ keys */

/* A14: SplitMix64 stream from the master seed; A = (next()>>32)|1, K_bh = next(). */
static uint64_t sm64_next(uint64_t* st) {
  uint64_t z = (*st += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* A^{-1} mod 2^32 by the extended Euclidean algorithm (A8; "A^{-1}*A=1 mod p"). */
static uint32_t inverse_mod_2_32(uint32_t A) {
  int64_t old_r = (int64_t)A, r = (int64_t)4294967296LL;
  int64_t old_s = 1, s = 0;
  while (r != 0) {
    int64_t q = old_r / r, tmp;
    tmp = old_r - q * r; old_r = r; r = tmp;
    tmp = old_s - q * s; old_s = s; s = tmp;
  }
  /* old_r == gcd == 1 for odd A; old_s * A == 1 (mod 2^32) */
  int64_t m = old_s % 4294967296LL;
  if (m < 0) m += 4294967296LL;
  return (uint32_t)m;
}

/* ----------------------------------------------------------- AT algebra */

/* Alg. 1 checkAT(at, k'), with act the ACT of the AT's block. */
int oracle_check_at(uint32_t at, uint32_t act, uint32_t k, uint32_t k_prime) {
  if (at == 2 * k) return 0;
  uint32_t dis = (act + 2 * k - at) % (2 * k);
  return dis <= k_prime - 1 ? 1 : 0;
}

/* Alg. 2 preserveAT(at). Returns the new value. */
uint32_t oracle_preserve_at(uint32_t at, uint32_t act, uint32_t k) {
  if ((act % k) != 0) return at;
  if (act == 0) {
    if (at <= k) at = 2 * k;                        /* P:227-228 (0 <= at <= k) */
  }
  if (act == k) {
    if (k <= at && at <= 2 * k - 1) at = 2 * k;
    if (at == 0) at = 2 * k;
  }
  return at;
}

/* Eq. 3 (A1): |OP| = -g ln((g - w)/g). */
double oracle_eq3(uint32_t w, uint32_t g) {
  return -(double)g * log((double)(g - w) / (double)g);
}

/* Eq. 5 (A19 brace reading): -g ln((g - NAT) / (g (1 - UP))), NAT real-valued. */
double oracle_eq5_real(double nat, double up, uint32_t g) {
  double num = (double)g - nat;
  double den = (double)g * (1.0 - up);
  return -(double)g * log(num / den);
}
/* Eq. 5 on the integer NAT of Alg. 5; NAT == g -> +inf (A20). */
double oracle_eq5(uint32_t nat, double up, uint32_t g) {
  if (nat == g) return INFINITY;
  return oracle_eq5_real((double)nat, up, g);
}

/* Super-ATV weight threshold |ATV|^{k'}_theta = g - g e^{-theta/g}. */
double oracle_w_theta(uint32_t g, double theta) {
  return (double)g - (double)g * exp(-theta / (double)g);
}

/* ------------------------------------------------------------ ATV blocks */

/* P:256 / A7: a = floor(g/2k), b = g - a(2k-1); AT i lies in block
 * min(i/a, 2k-1) (all in block 2k-1 when a = 0); block clock (C0+i) mod 2k. */
static uint32_t block_of(const oracle_t* o, uint32_t i) {
  uint32_t two_k = 2 * o->p.k;
  if (o->a == 0) return two_k - 1;
  uint32_t bl = i / o->a;
  return bl < two_k - 1 ? bl : two_k - 1;
}
uint32_t oracle_block(const oracle_t* o, uint32_t i) { return block_of(o, i); }
uint32_t oracle_act(const oracle_t* o, uint32_t i) {
  return (o->C0 + block_of(o, i)) % (2 * o->p.k);
}

/* ------------------------------------------------------------------ RRH */

#define MANGLE_P 4294967311ULL   /* the smallest prime above 2^32 */

static uint64_t mulmod_p(uint64_t a, uint64_t b) {
  return (uint64_t)(((unsigned __int128)a * b) % MANGLE_P);
}
/* f(aip) = A * aip mod 2^32 (A8), or — SURVEY §8(f) row 4, the paper-literal form —
 * f(aip) = A * aip mod p with p prime > 2^32. The latter is a bijection of
 * [0, p); the values >= 2^32 it yields for 32-bit inputs are stepped through f again
 * (cycle walking) until they fit in 32 bits, which keeps f a bijection of [0, 2^32). */
uint32_t oracle_mangle(const oracle_t* o, uint32_t ip) {
  if (!o->p.mangle) return (uint32_t)(o->A * ip);
  uint64_t y = mulmod_p(o->A, ip);
  while (y >= 4294967296ULL) y = mulmod_p(o->A, y);
  return (uint32_t)y;
}
/* f^{-1}(h) = A^{-1} h ("aip could be regain by f^{-1}"), walked the same way. */
uint32_t oracle_unmangle(const oracle_t* o, uint32_t h) {
  if (!o->p.mangle) return (uint32_t)(o->A_inv * h);
  uint64_t x = mulmod_p(o->A_inv, h);
  while (x >= 4294967296ULL) x = mulmod_p(o->A_inv, x);
  return (uint32_t)x;
}

/* Z(aip) = RBS(f(aip), u); LBS = the left 32-u bits, LBS[p] its p-th bit
 * counted from the least significant end (A9); x_y[j] = LBS[(s*y + j) mod (32-u)]
 * ("successive c bits starting from s*i ... loop to starting from 0"). */
void oracle_digest(const oracle_t* o, uint32_t ip, uint32_t* z, uint32_t* x) {
  const uint32_t u = o->p.u, c = o->p.c, s = o->p.s, W = 32 - u;
  uint32_t h = oracle_mangle(o, ip);
  uint32_t lbs = (u == 32) ? 0 : (h >> u);
  *z = (u == 0) ? 0 : (h & ((1u << u) - 1u));
  for (uint32_t y = 0; y < o->p.r; ++y) {
    uint32_t xy = 0;
    for (uint32_t j = 0; j < c; ++j) {
      uint32_t pos = (s * y + j) % W;
      uint32_t bit = (lbs >> pos) & 1u;
      xy |= bit << j;
    }
    x[y] = xy;
  }
}

/* BH(bip) in [0, g) (A13): ((SplitMix64-finalizer(bip ^ K_bh) >> 32) * g) >> 32 */
uint32_t oracle_bh(const oracle_t* o, uint32_t bip) {
  uint64_t z = (uint64_t)bip ^ o->K_bh;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z = z ^ (z >> 31);
  return (uint32_t)(((z >> 32) * (uint64_t)o->p.g) >> 32);
}

/* Alg. 4: concatenate the sub bits of <x_0..x_{r-1}> into the LBS,
 * after checking every duplicate position agrees (all pairs, A16).
 * Returns 1 and the LBS when consistent, 0 otherwise. */
int oracle_restore_lbs(const oracle_t* o, const uint32_t* x, uint32_t* lbs_out) {
  const uint32_t c = o->p.c, s = o->p.s, W = 32 - o->p.u;
  uint32_t lbs = 0;
  uint8_t known[32] = {0};
  for (uint32_t y = 0; y < o->p.r; ++y) {
    for (uint32_t j = 0; j < c; ++j) {
      uint32_t pos = (s * y + j) % W;
      uint32_t bit = (x[y] >> j) & 1u;
      if (known[pos]) {
        if (((lbs >> pos) & 1u) != bit) return 0;
      } else {
        known[pos] = 1;
        lbs |= bit << pos;
      }
    }
  }
  *lbs_out = lbs;
  return 1;
}
/* Alg. 4: randip = LBS||RBS with RBS = frame j; sip = f^{-1}(randip). */
uint32_t oracle_restore_ip(const oracle_t* o, uint32_t lbs, uint32_t z) {
  uint32_t randip = (o->p.u == 32 ? 0 : (lbs << o->p.u)) | z;
  return oracle_unmangle(o, randip);
}

/* -------------------------------------------------------------- lifecycle */

static size_t atv_index(const oracle_t* o, uint32_t y, uint32_t z, uint32_t x) {
  return ((size_t)y * o->F + z) * o->E + x;
}
static size_t at_index(const oracle_t* o, uint32_t y, uint32_t z, uint32_t x, uint32_t i) {
  return atv_index(o, y, z, x) * o->p.g + i;
}

/* Completeness / redundancy attributes (A10). */
int oracle_validate(const oracle_params* p, char* why, size_t n) {
#define BAD(msg) do { if (why && n) snprintf(why, n, "%s", msg); return ORACLE_E_PARAM; } while (0)
  if (p->k < 1) BAD("k >= 1");
  if (p->k_prime < 1 || p->k_prime > p->k) BAD("1 <= k' <= k");
  if (p->g < 1) BAD("g >= 1");
  if (p->r < 2) BAD("r >= 2");
  if (p->u > 31 || p->c < 1 || p->c + p->u > 32) BAD("c >= 1, u <= 31, c + u <= 32");
  if (p->s < 1 || p->s > p->c) BAD("1 <= s <= c");
  if (!(p->theta > 0)) BAD("theta > 0");
  if (p->mangle > 1) BAD("mangle is 0 or 1");
  uint32_t W = 32 - p->u;
  if (p->c + p->s * (p->r - 1) < W) BAD("completeness: c + s(r-1) >= 32-u");
  uint32_t cover[32] = {0};
  for (uint32_t y = 0; y < p->r; ++y)
    for (uint32_t j = 0; j < p->c; ++j) cover[(p->s * y + j) % W]++;
  int dup = 0;
  for (uint32_t q = 0; q < W; ++q) {
    if (cover[q] == 0) BAD("completeness: a LBS bit is not covered");
    if (cover[q] >= 2) dup = 1;
  }
  if (!dup) BAD("redundancy: no duplicate position");
  return ORACLE_OK;
#undef BAD
}

oracle_t* oracle_new(const oracle_params* p, char* why, size_t n) {
  if (oracle_validate(p, why, n) != ORACLE_OK) return NULL;
  oracle_t* o = (oracle_t*)calloc(1, sizeof(oracle_t));
  o->p = *p;
  o->F = 1u << p->u;
  o->E = 1u << p->c;
  o->a = p->g / (2 * p->k);
  o->b = p->g - o->a * (2 * p->k - 1);
  uint64_t st = p->seed;
  if (!p->mangle) {
    o->A = (uint32_t)(sm64_next(&st) >> 32) | 1u;
    o->K_bh = sm64_next(&st);
    o->A_inv = inverse_mod_2_32((uint32_t)o->A);
  } else {
    /* A uniform in [1, p-1]; A^{-1} = A^{p-2} mod p (Fermat) */
    o->A = sm64_next(&st) % (MANGLE_P - 1) + 1;
    o->K_bh = sm64_next(&st);
    uint64_t r = 1, b = o->A, e = MANGLE_P - 2;
    while (e) { if (e & 1) r = mulmod_p(r, b); b = mulmod_p(b, b); e >>= 1; }
    o->A_inv = r;
  }
  size_t n_atv = (size_t)p->r * o->F * o->E;
  size_t n_at = n_atv * p->g;
  o->pool = (uint16_t*)malloc(n_at * sizeof(uint16_t));
  o->w = (uint32_t*)calloc(n_atv, sizeof(uint32_t));
  o->super = (uint8_t*)calloc(n_atv, 1);
  o->aat = (uint64_t*)calloc((size_t)p->r * o->F, sizeof(uint64_t));
  if (!o->pool || !o->w || !o->super || !o->aat) {
    if (why && n) snprintf(why, n, "out of memory");
    free(o->pool); free(o->w); free(o->super); free(o->aat); free(o);
    return NULL;
  }
  /* step 0: InitAT every AT; C0 = 0, t = 0 (A3) */
  for (size_t q = 0; q < n_at; ++q) o->pool[q] = (uint16_t)(2 * p->k);
  o->C0 = 0;
  o->t = 0;
  return o;
}

void oracle_free(oracle_t* o) {
  if (!o) return;
  free(o->pool); free(o->w); free(o->super); free(o->aat); free(o->rep);
  free(o);
}

void oracle_keys(const oracle_t* o, uint64_t* A, uint64_t* A_inv, uint64_t* K_bh) {
  *A = o->A; *A_inv = o->A_inv; *K_bh = o->K_bh;
}
void oracle_blocks(const oracle_t* o, uint32_t* a, uint32_t* b) { *a = o->a; *b = o->b; }
uint32_t oracle_C0(const oracle_t* o) { return o->C0; }
uint64_t oracle_slice(const oracle_t* o) { return o->t; }
uint64_t oracle_pool_size(const oracle_t* o) {
  return (uint64_t)o->p.r * o->F * o->E * o->p.g;
}

/* ------------------------------------------------------------- step 1 */

/* SetAT on one AT: value := ACT of its block. Used by Alg. 3 and tests. */
void oracle_touch(oracle_t* o, uint32_t y, uint32_t z, uint32_t x, uint32_t i) {
  o->pool[at_index(o, y, z, x, i)] = (uint16_t)oracle_act(o, i);
}

/* Alg. 3 "Scan IP pair" for each pair of slice t. */
void oracle_scan(oracle_t* o, const uint32_t* pairs, uint64_t n) {
  uint32_t x[32], z;
  for (uint64_t q = 0; q < n; ++q) {
    uint32_t aip = pairs[2 * q], bip = pairs[2 * q + 1];   /* A33: first u32 is aip */
    oracle_digest(o, aip, &z, x);                          /* RRH(aip) */
    uint32_t i = oracle_bh(o, bip);
    for (uint32_t y = 0; y < o->p.r; ++y)
      oracle_touch(o, y, z, x[y], i);                      /* P:347 SetAT */
  }
}

/* The same Alg. 3 loop split over host threads — used ONLY by bench.py's optional
 * all-core CPU baseline (SURVEY §8(d) "Oracle timing"), never for parity. Every SetAT of
 * slice t writes the ACT of its block, a value fixed by (i, C0), so concurrent
 * writers of one AT store the same value: relaxed atomic stores give the pool of
 * oracle_scan exactly (pinned by tests/test_oracle_scan_mt.py). nthreads <= 0: every core. */
void oracle_scan_mt(oracle_t* o, const uint32_t* pairs, uint64_t n, int nthreads) {
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
  {
    uint32_t x[32], z;
#pragma omp for schedule(static)
    for (uint64_t q = 0; q < n; ++q) {
      uint32_t aip = pairs[2 * q], bip = pairs[2 * q + 1];
      oracle_digest(o, aip, &z, x);
      uint32_t i = oracle_bh(o, bip);
      uint16_t v = (uint16_t)oracle_act(o, i);
      for (uint32_t y = 0; y < o->p.r; ++y)
        __atomic_store_n(&o->pool[at_index(o, y, z, x[y], i)], v, __ATOMIC_RELAXED);
    }
  }
#else
  (void)nthreads;
  oracle_scan(o, pairs, n);
#endif
}

int oracle_omp_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------- steps 2-6 */

static int cmp_report(const void* a, const void* b) {
  uint32_t x = ((const oracle_report*)a)->ip, y = ((const oracle_report*)b)->ip;
  return (x > y) - (x < y);
}

/* Alg. 5 NAT(aip): number of i active in all r ATVs of aip. */
uint32_t oracle_nat(const oracle_t* o, uint32_t aip) {
  uint32_t x[32], z;
  oracle_digest(o, aip, &z, x);
  uint32_t nat = 0;
  for (uint32_t i = 0; i < o->p.g; ++i) {
    int active = 1;
    uint32_t act = oracle_act(o, i);
    for (uint32_t j = 0; j < o->p.r; ++j) {
      uint32_t at = o->pool[at_index(o, j, z, x[j], i)];
      if (!oracle_check_at(at, act, o->p.k, o->p.k_prime)) { active = 0; break; }
    }
    if (active) nat++;
  }
  return nat;
}

typedef struct {
  oracle_t* o;
  uint32_t z;
  uint32_t** sa;    /* SA(y, z) lists */
  uint32_t* n_sa;
  int overflow;
} restore_ctx;

static int add_report(oracle_t* o, uint32_t ip) {
  if (o->n_rep >= o->p.max_candidates) return ORACLE_E_OVERFLOW;
  if (o->n_rep == o->cap_rep) {
    uint32_t nc = o->cap_rep ? 2 * o->cap_rep : 1024;
    oracle_report* r = (oracle_report*)realloc(o->rep, nc * sizeof(oracle_report));
    if (!r) return ORACLE_E_OVERFLOW;
    o->rep = r;
    o->cap_rep = nc;
  }
  o->rep[o->n_rep].ip = ip;
  o->rep[o->n_rep].nat = 0;
  o->rep[o->n_rep].estimate = 0;
  o->rep[o->n_rep].flags = 0;
  o->rep[o->n_rep].pad = 0;
  o->n_rep++;
  return ORACLE_OK;
}

/* Alg. 4 line 364 (product over rows) with the line 365-369 duplicate-position
 * check applied as soon as row y is assigned (A16: same set). */
static void restore_rows(restore_ctx* rc, uint32_t y, uint32_t lbs, const uint8_t* known) {
  oracle_t* o = rc->o;
  if (rc->overflow) return;
  if (y == o->p.r) {
    uint32_t ip = oracle_restore_ip(o, lbs, rc->z);
    if (add_report(o, ip) != ORACLE_OK) rc->overflow = 1;  /* P:374 Insert sip */
    return;
  }
  const uint32_t c = o->p.c, s = o->p.s, W = 32 - o->p.u;
  for (uint32_t q = 0; q < rc->n_sa[y]; ++q) {
    uint32_t x = rc->sa[y][q];
    uint32_t nl = lbs;
    uint8_t nk[32];
    memcpy(nk, known, 32);
    int ok = 1;
    for (uint32_t j = 0; j < c && ok; ++j) {
      uint32_t pos = (s * y + j) % W;
      uint32_t bit = (x >> j) & 1u;
      if (nk[pos]) {
        if (((nl >> pos) & 1u) != bit) ok = 0;   /* duplicate position disagrees */
      } else {
        nk[pos] = 1;
        nl |= bit << pos;
      }
    }
    if (ok) restore_rows(rc, y + 1, nl, nk);
  }
}

/* Steps 2-6 for the current slice t; results stay in o->rep (ascending ip). */
int oracle_detect(oracle_t* o) {
  const oracle_params* p = &o->p;
  const uint32_t g = p->g;
  const double w_theta = oracle_w_theta(g, p->theta);
  o->n_rep = 0;
  /* step 2: |ATV|^{k'} = number of active ATs, AAT */
  for (uint32_t y = 0; y < p->r; ++y)
    for (uint32_t z = 0; z < o->F; ++z) {
      uint64_t aat = 0;
      for (uint32_t x = 0; x < o->E; ++x) {
        uint32_t w = 0;
        for (uint32_t i = 0; i < g; ++i)
          w += (uint32_t)oracle_check_at(o->pool[at_index(o, y, z, x, i)], oracle_act(o, i),
                                         p->k, p->k_prime);
        o->w[atv_index(o, y, z, x)] = w;
        /* step 3: super ATV iff |ATV|^{k'} no smaller than the threshold */
        o->super[atv_index(o, y, z, x)] = ((double)w >= w_theta) ? 1 : 0;
        aat += w;
      }
      o->aat[(size_t)y * o->F + z] = aat;
    }
  /* step 4: Alg. 4 frame by frame (frames 0..2^u-1, A16) */
  uint32_t** sa = (uint32_t**)calloc(p->r, sizeof(uint32_t*));
  uint32_t* n_sa = (uint32_t*)calloc(p->r, sizeof(uint32_t));
  for (uint32_t y = 0; y < p->r; ++y) sa[y] = (uint32_t*)malloc(o->E * sizeof(uint32_t));
  int rc_status = ORACLE_OK;
  for (uint32_t z = 0; z < o->F && rc_status == ORACLE_OK; ++z) {
    for (uint32_t y = 0; y < p->r; ++y) {
      n_sa[y] = 0;
      for (uint32_t x = 0; x < o->E; ++x)
        if (o->super[atv_index(o, y, z, x)]) sa[y][n_sa[y]++] = x;  /* SA(y, z) */
    }
    restore_ctx rc = {o, z, sa, n_sa, 0};
    uint8_t known[32] = {0};
    restore_rows(&rc, 0, 0, known);
    if (rc.overflow) rc_status = ORACLE_E_OVERFLOW;
  }
  for (uint32_t y = 0; y < p->r; ++y) free(sa[y]);
  free(sa);
  free(n_sa);
  if (rc_status != ORACLE_OK) return rc_status;
  /* step 5: NAT (Alg. 5), UP (Eq. 4 / P:412), estimate (Eq. 5) */
  const double cells = (double)g * (double)o->E;     /* g * 2^c */
  for (uint32_t q = 0; q < o->n_rep; ++q) {
    oracle_report* R = &o->rep[q];
    uint32_t x[32], z;
    oracle_digest(o, R->ip, &z, x);
    R->nat = oracle_nat(o, R->ip);
    double up = 0.0;
    for (uint32_t y = 0; y < p->r; ++y) {
      double P = (double)o->aat[(size_t)y * o->F + z] / cells;   /* P_{y,z}^{k'} */
      up = (y == 0) ? P : up * P;                                 /* UP = prod_y P */
    }
    R->estimate = oracle_eq5(R->nat, up, g);
    R->flags = (R->nat == g ? 1u : 0u) | (R->estimate >= p->theta ? 2u : 0u);
  }
  /* step 6: ascending ip (A24) */
  qsort(o->rep, o->n_rep, sizeof(oracle_report), cmp_report);
  return ORACLE_OK;
}

/* ------------------------------------------------------------- step 7 */

/* ACT advances by one per slice; preserveAT at the beginning of the
 * new slice on every AT, i.e. Alg. 2 with its ACT (A3, A32). */
void oracle_advance(oracle_t* o) {
  const oracle_params* p = &o->p;
  o->t += 1;
  o->C0 = (uint32_t)(o->t % (2 * p->k));
  size_t n_atv = (size_t)p->r * o->F * o->E;
  for (uint32_t i = 0; i < p->g; ++i) {
    uint32_t act = oracle_act(o, i);
    if (act % p->k != 0) continue;  /* Alg. 2 line 223 early return, hoisted per block */
    for (size_t v = 0; v < n_atv; ++v) {
      uint16_t* at = &o->pool[v * p->g + i];
      *at = (uint16_t)oracle_preserve_at(*at, act, p->k);
    }
  }
}

/* end_slice(t): detect at t, copy reports (mode 0: est >= theta; mode 1: all CSIP),
 * then advance to t+1. Returns ORACLE_E_CAPACITY with *n_out = needed if cap is small. */
int oracle_end_slice(oracle_t* o, int mode, oracle_report* out, uint32_t cap, uint32_t* n_out) {
  int st = oracle_detect(o);
  if (st != ORACLE_OK) { oracle_advance(o); *n_out = 0; return st; }
  uint32_t n = 0;
  for (uint32_t q = 0; q < o->n_rep; ++q)
    if (mode == 1 || (o->rep[q].flags & 2u)) {
      if (out && n < cap) out[n] = o->rep[q];
      n++;
    }
  *n_out = n;
  oracle_advance(o);
  return (out && n > cap) ? ORACLE_E_CAPACITY : ORACLE_OK;
}

/* ------------------------------------------------------------ accessors */

void oracle_export_pool(const oracle_t* o, uint16_t* out) {
  memcpy(out, o->pool, oracle_pool_size(o) * sizeof(uint16_t));
}
void oracle_import_pool(oracle_t* o, const uint16_t* in) {
  memcpy(o->pool, in, oracle_pool_size(o) * sizeof(uint16_t));
}
void oracle_weights(const oracle_t* o, uint32_t* w, uint64_t* aat, uint8_t* super) {
  size_t n_atv = (size_t)o->p.r * o->F * o->E;
  if (w) memcpy(w, o->w, n_atv * sizeof(uint32_t));
  if (aat) memcpy(aat, o->aat, (size_t)o->p.r * o->F * sizeof(uint64_t));
  if (super) memcpy(super, o->super, n_atv);
}
uint32_t oracle_n_reports(const oracle_t* o) { return o->n_rep; }
void oracle_reports(const oracle_t* o, oracle_report* out) {
  memcpy(out, o->rep, (size_t)o->n_rep * sizeof(oracle_report));
}

/* ---------------------------------------------------- multi-pool combine */

/* A26 (paper silent): most-recent-wins combine of D pools that
 * share one clock: per AT keep the value with the smallest age (act - v) mod 2k,
 * inactive (2k) counting as infinitely old. Result written to `out`. */
void oracle_combine_min_age(const oracle_t* o, const uint16_t* const* pools, uint32_t D,
                            uint16_t* out) {
  const uint32_t two_k = 2 * o->p.k;
  size_t n_atv = (size_t)o->p.r * o->F * o->E;
  for (uint32_t i = 0; i < o->p.g; ++i) {
    uint32_t act = oracle_act(o, i);
    for (size_t v = 0; v < n_atv; ++v) {
      size_t q = v * o->p.g + i;
      uint32_t best = two_k, best_age = 0xFFFFFFFFu;
      for (uint32_t d = 0; d < D; ++d) {
        uint32_t val = pools[d][q];
        if (val == two_k) continue;
        uint32_t age = (act + two_k - val) % two_k;
        if (age < best_age) { best_age = age; best = val; }
      }
      out[q] = (uint16_t)best;
    }
  }
}
