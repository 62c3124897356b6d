/*
 * truth.c — exact sliding-window cardinality oracle (TEST INFRASTRUCTURE).
 *
 * |OP(aip, W)| = number of distinct bip seen with aip in the window of the
 * last k' slices (window semantics P:115, A4, A35). Super point iff
 * |OP| >= theta (A22). Used only to report FPR / FNR / MRE (Def. 1,
 * P:448-452) and to pin the ASSE oracle on tiny traces. Shares nothing with
 * the ASSE oracle or the CUDA path.
 *
 * Data structure: open-addressing hash map pair -> last slice seen; per-aip
 * hash map aip -> count of pairs whose last slice is inside the window; one
 * list per slice of pairs (re)stamped in that slice, used to expire them.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { uint64_t* key; uint32_t* val; uint64_t cap, n; } hmap; /* key 0 = empty */

static uint64_t hmix(uint64_t x) {
  x ^= x >> 31; x *= 0x7fb5d329728ea185ULL; x ^= x >> 27; x *= 0x81dadef4bc2dd44dULL;
  return x ^ (x >> 33);
}
static void hm_init(hmap* m, uint64_t cap) {
  m->cap = cap; m->n = 0;
  m->key = (uint64_t*)calloc(cap, 8);
  m->val = (uint32_t*)calloc(cap, 4);
}
static uint32_t* hm_find(hmap* m, uint64_t k, int insert);
static void hm_grow(hmap* m) {
  hmap nm;
  hm_init(&nm, m->cap * 2);
  for (uint64_t q = 0; q < m->cap; ++q)
    if (m->key[q]) *hm_find(&nm, m->key[q] - 1, 1) = m->val[q];
  free(m->key); free(m->val);
  *m = nm;
}
/* keys are stored +1 so that 0 marks empty */
static uint32_t* hm_find(hmap* m, uint64_t k, int insert) {
  if (insert && 2 * (m->n + 1) > m->cap) hm_grow(m);
  uint64_t kk = k + 1, q = hmix(kk) & (m->cap - 1);
  while (m->key[q]) {
    if (m->key[q] == kk) return &m->val[q];
    q = (q + 1) & (m->cap - 1);
  }
  if (!insert) return NULL;
  m->key[q] = kk; m->val[q] = 0; m->n++;
  return &m->val[q];
}

typedef struct { uint64_t* v; uint64_t n, cap; } vec;
static void vec_push(vec* a, uint64_t x) {
  if (a->n == a->cap) { a->cap = a->cap ? 2 * a->cap : 1024; a->v = (uint64_t*)realloc(a->v, a->cap * 8); }
  a->v[a->n++] = x;
}

typedef struct {
  uint32_t k_prime;
  int64_t t;            /* current slice index (-1 before the first) */
  hmap last;            /* pair -> last slice + 1 */
  hmap count;           /* aip -> in-window distinct peers */
  vec* lists;           /* ring of k'+1 per-slice lists */
} truth_t;

truth_t* truth_new(uint32_t k_prime) {
  truth_t* T = (truth_t*)calloc(1, sizeof(truth_t));
  T->k_prime = k_prime;
  T->t = -1;
  hm_init(&T->last, 1u << 20);
  hm_init(&T->count, 1u << 16);
  T->lists = (vec*)calloc(k_prime + 1, sizeof(vec));
  return T;
}
void truth_free(truth_t* T) {
  if (!T) return;
  free(T->last.key); free(T->last.val); free(T->count.key); free(T->count.val);
  for (uint32_t q = 0; q <= T->k_prime; ++q) free(T->lists[q].v);
  free(T->lists); free(T);
}

/* Begin slice t+1: expire pairs whose last sighting is slice t+1-k'. */
void truth_begin_slice(truth_t* T) {
  T->t += 1;
  int64_t old = T->t - (int64_t)T->k_prime;
  vec* L = &T->lists[T->t % (T->k_prime + 1)];
  if (old >= 0) {
    vec* E = &T->lists[old % (T->k_prime + 1)];
    for (uint64_t q = 0; q < E->n; ++q) {
      uint32_t* lv = hm_find(&T->last, E->v[q], 0);
      if (lv && (int64_t)*lv - 1 == old) {
        uint32_t* c = hm_find(&T->count, E->v[q] >> 32, 0);
        if (c) (*c)--;
      }
    }
    E->n = 0;
  }
  L->n = 0;
}

void truth_add(truth_t* T, const uint32_t* pairs, uint64_t n) {
  for (uint64_t q = 0; q < n; ++q) {
    uint64_t key = ((uint64_t)pairs[2 * q] << 32) | pairs[2 * q + 1];
    uint32_t* lv = hm_find(&T->last, key, 1);
    int64_t last = (int64_t)*lv - 1;           /* -1 if new */
    if (last == T->t) continue;                /* already stamped this slice */
    if (last < 0 || last <= T->t - (int64_t)T->k_prime)  /* new or expired: enters window */
      (*hm_find(&T->count, key >> 32, 1))++;
    *lv = (uint32_t)(T->t + 1);
    vec_push(&T->lists[T->t % (T->k_prime + 1)], key);
  }
}

uint32_t truth_card(truth_t* T, uint32_t aip) {
  uint32_t* c = hm_find(&T->count, aip, 0);
  return c ? *c : 0;
}

/* aips with window cardinality >= theta; returns the count, fills up to cap. */
uint64_t truth_supers(truth_t* T, uint32_t theta, uint32_t* out, uint32_t* card, uint64_t cap) {
  uint64_t n = 0;
  for (uint64_t q = 0; q < T->count.cap; ++q)
    if (T->count.key[q] && T->count.val[q] >= theta) {
      if (n < cap) { out[n] = (uint32_t)(T->count.key[q] - 1); if (card) card[n] = T->count.val[q]; }
      n++;
    }
  return n;
}
