// asse_scan_own.cuh — Alg. 3 with packet-granular ownership of the touch bitmap.
//
// k_scan_bin (asse_scan_bin.cuh) bins each of a packet's r SetATs separately: r targets
// computed by the producer, r slot atomics, r 4-byte queue entries and one row through
// L2 REDs. Here the unit that travels is the PACKET, not the SetAT. A host's r ATVs share
// its frame z = f(aip) mod 2^u and all r SetATs of a packet hit the same AT
// position i = BH(bip) (Alg. 3 computes i once). So the pair (z, word group of i) names a
// slice of the bitmap that holds all r targets of the packet:
//
//   owner o = z * NGRP + (i >> 5) / WG       (NGRP word groups of WG words per ATV)
//   slice(o) = rows 0..r-1, the 2^c ATVs of frame z, words [grp*WG, (grp+1)*WG) of each
//
// At the C3-C5 geometry (F = 16 frames, 2^c = 4096, g = 512: 16 words per ATV) NGRP = 8,
// WG = 2: 128 owners of 128 KiB each. The producer computes f(aip) and BH(bip), takes one
// slot in the owner's bin and stores an 8-byte entry (L, word, touch mask); the owner derives the r
// column windows itself and applies the r SetATs with shared-memory atomics.
// Per packet: 1 slot atomic (k_scan_bin: 3), 8 B through the L2 queues (12 B + a RED), no
// global RED. CTAs beyond the O owners produce only.
//
// Round structure, queues, publication and drain are k_scan_bin's; the
// touch bits after the call are the same union (SetAT is idempotent within a slice),
// so the pool after every slice is bit-identical to k_scan's and the oracle's.
#pragma once
#include "asse_scan_bin.cuh"

// ASSE_OWN_DEBUG_BOUNDS=1: device asserts on every index the kernel derives (owner, slot,
// slice word, ring ranges, write-back word) — the bounds check used on the GPU pool, where
// compute-sanitizer is unavailable (tools/gpu_own_bounds.sh runs the parity tests with it)
#ifndef ASSE_OWN_DEBUG_BOUNDS
#define ASSE_OWN_DEBUG_BOUNDS 0
#endif
#if ASSE_OWN_DEBUG_BOUNDS
#include <cassert>
#define OWN_ASSERT(x) assert(x)
#else
#define OWN_ASSERT(x) ((void)0)
#endif

namespace asse {

#ifndef ASSE_OWN_BIN_WARPS
#define ASSE_OWN_BIN_WARPS 8
#endif
#ifndef ASSE_OWN_CONS_WARPS
#define ASSE_OWN_CONS_WARPS 8
#endif
#ifndef ASSE_OWN_NB
#define ASSE_OWN_NB 8
#endif
#ifndef ASSE_OWN_NGR
#define ASSE_OWN_NGR 4
#endif
#ifndef ASSE_OWN_U
#define ASSE_OWN_U 1
#endif
// warps (measured at C5 on B200, tools/gpu_own_sweep2.sh, gpu_own13.sh): with runtime geometry
// 16 binning + 8 / 10 / 12 / 14 draining warps 0.98 / 1.07 / 0.94 / 0.95 ms; with the C3
// geometry folded (cheaper drain) 6 / 8 / 10 / 12 warps 0.95 / 0.82 / 0.86 / 0.84 ms, 8 warps
// with two 16-B groups in flight per ring 0.81 ms. Binning warps (8 draining, 6 rings, one 16-B
// group in flight, tools/gpu_own28-30.sh): 16 / 14 / 12 / 10 / 8 / 6 / 4 warps 0.79 / 0.79 /
// 0.77 / 0.82 / 0.74 / 0.89 / 1.32 ms — fewer warps leave each thread more registers (96 at
// 8 warps: no address rematerialisation in the binning loop); 8 warps with 6 or 12 draining
// warps 0.86 / 1.16 ms
constexpr int kOwnBinWarps = ASSE_OWN_BIN_WARPS;           // binning + shipping warps
constexpr int kOwnConsWarps = ASSE_OWN_CONS_WARPS;         // queue-draining warps, two groups (round parity)
constexpr int kOwnConsWarp0 = kOwnBinWarps;
constexpr int kOwnTmaWarp = kOwnConsWarp0 + kOwnConsWarps;
constexpr int kOwnSigWarp = kOwnTmaWarp + 1;
// buffer-reuse handoff (the global acquire of cons_done, see the free loop below) runs in
// lane 1 of the TMA warp. Alternatives measured at C5 (scan ms, tools/sweep.py r02k-r02n;
// round 1's relaxed probes without any acquire: 0.715): the binning warps probing cons_done
// with an acquire themselves 0.754 (the acquire stalls the round); a warp of its own 0.755
// (ptxas drops to 92 registers and the binning loop rematerialises); lane 1 of the signal
// warp 0.750; lane 1 of the TMA warp 0.729.
constexpr int kOwnThreads = 32 * (kOwnSigWarp + 1);
constexpr int kOwnRing = 2;                                // packet-tile ring stages
constexpr uint32_t kOwnCap = 30;                           // staged entries per (owner, round) in a CTA; also
                                                           // the bin stride (240 B, 16-B aligned; bin o
                                                           // starts at bank 28o mod 32)
constexpr uint32_t kOwnNB = ASSE_OWN_NB;                   // queue buffers (rounds) in flight (C5: 4 -> 0.952 ms,
                                                           // 6 0.942, 8 0.927; tools/gpu_own_sweep4.sh)
constexpr uint32_t kOwnNGR = ASSE_OWN_NGR;                 // drain groups (round t -> group t mod NGR)
static_assert(kOwnNB % kOwnNGR == 0 && kOwnConsWarps % kOwnNGR == 0, "drain groups");
static_assert(2 + kOwnNGR <= 8, "named barriers 2 .. 1 + NGR must stay below the compute barrier 8");
// drain groups (8 binning / 8 draining warps, tools/gpu_own32-33.sh): 1 / 2 / 4 groups
// 0.966 / 0.739 / 0.716 ms at C5
#ifndef ASSE_OWN_QG
#define ASSE_OWN_QG 6
#endif
constexpr uint32_t kOwnQG = ASSE_OWN_QG;                   // producer groups (CTA index mod QG), one ring each
                                                           // per (buffer, owner): C5 2 / 4 / 6 / 8 groups
                                                           // 0.807 / 0.795 / 0.791 / 1.22 ms
#ifndef ASSE_OWN_QCAP
#define ASSE_OWN_QCAP 1024
#endif
constexpr uint32_t kOwnQCap = ASSE_OWN_QCAP;
static_assert((kOwnQCap & (kOwnQCap - 1)) == 0, "ring index is masked");                        // ring entries per (buffer, owner, group) >= the
                                                           // producer group's bins (host-checked)

#ifndef OWN_FREE_SLEEP
#define OWN_FREE_SLEEP 256
#endif
constexpr uint32_t kOwnMaxOwners = 128;                   // F * NGRP: a power of two <= the SMs
constexpr uint32_t kOwnMinTilesPerCta = 8;                 // below: k_scan is used

struct OwnScanParams {
  ScanParams sp;          // hashing parameters and the global touch bitmap
  uint2* queue;           // [NB][O][QG][QCAP] rings of entries (see own_bin_two)
  uint32_t* qcnt;         // [NB][O][QG] x kBinPad: entries ever reserved (monotone per launch)
  uint32_t* sync;         // [2 NB] x kBinPad: rounds published per buffer, then owners done; zero at launch
  uint32_t* sync_next;    // the other counter set (sync + qcnt of the next launch): zeroed here
  uint32_t sync_words;
  uint32_t O;             // owners = F << lg_ngrp (<= gridDim.x)
  uint32_t lg_ngrp;       // word groups per ATV (log2)
  uint32_t lg_wg;         // words per group (log2)
  uint32_t tile_bytes;    // packets per CTA per round x 8
  unsigned long long* prof;  // optional per-CTA phase cycle counters [G][16] (tools; may be null)
};

// dynamic shared memory: [ring 2 tiles][staging 2 x O x CAP][counts][owners: the slice]
__host__ __device__ constexpr size_t own_smem_bytes(uint32_t O, uint32_t slice_words, uint32_t tile_bytes) {
  return (size_t)kOwnRing * tile_bytes + 2 * (size_t)O * kOwnCap * 8 + 2 * (((size_t)O * 4 + 15) & ~(size_t)15) +
         16 + (size_t)slice_words * 4;
}

// mbarrier wait for warps off the critical path: the hardware suspends the thread until
// the phase completes or the hint (ns) expires, so the wait costs no issue slots (a
// nanosleep poll loop cost ~8 % of the kernel's instructions, ncu r01g)
__device__ __forceinline__ void mbar_wait_suspend(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done) : "r"(smem_u32(bar)), "r"(phase), "r"(1000000u) : "memory");
  }
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void sts64_if(bool pred, uint32_t addr, uint32_t a, uint32_t b) {
  asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %0, 0;\n @p st.shared.v2.u32 [%1], {%2, %3};\n}"
               :: "r"((uint32_t)pred), "r"(addr), "r"(a), "r"(b) : "memory");
}

// Geometry seen by the hot loops: runtime values (any geometry own_ok admits) or
// compile-time constants for the BASELINE C3-C5 geometry (u = 4, c = 12, s = 6, g = 512,
// NGRP = 8, WG = 2), so shifts, masks and the column-window offsets fold into immediates
// (ncu r01h: the owner-side SetAT took 36 instructions per entry with runtime values).
struct GeoRt {
  __device__ static __forceinline__ uint32_t u(const OwnScanParams& op) { return op.sp.u; }
  __device__ static __forceinline__ uint32_t W(const OwnScanParams& op) { return op.sp.W; }
  __device__ static __forceinline__ uint32_t c(const OwnScanParams& op) { return op.sp.c; }
  __device__ static __forceinline__ uint32_t cmask(const OwnScanParams& op) { return op.sp.cmask; }
  __device__ static __forceinline__ uint32_t fmask(const OwnScanParams& op) { return op.sp.fmask; }
  __device__ static __forceinline__ uint32_t g(const OwnScanParams& op) { return op.sp.g; }
  __device__ static __forceinline__ uint32_t shift(const OwnScanParams& op, int y) { return op.sp.shift[y]; }
  __device__ static __forceinline__ uint32_t lg_ngrp(const OwnScanParams& op) { return op.lg_ngrp; }
  __device__ static __forceinline__ uint32_t lg_wg(const OwnScanParams& op) { return op.lg_wg; }
};
template <uint32_t U_, uint32_t C_, uint32_t S_, uint32_t G_, uint32_t LGNG_, uint32_t LGWG_>
struct GeoCt {
  __device__ static __forceinline__ constexpr uint32_t u(const OwnScanParams&) { return U_; }
  __device__ static __forceinline__ constexpr uint32_t W(const OwnScanParams&) { return 32u - U_; }
  __device__ static __forceinline__ constexpr uint32_t c(const OwnScanParams&) { return C_; }
  __device__ static __forceinline__ constexpr uint32_t cmask(const OwnScanParams&) { return (1u << C_) - 1u; }
  __device__ static __forceinline__ constexpr uint32_t fmask(const OwnScanParams&) { return (1u << U_) - 1u; }
  __device__ static __forceinline__ constexpr uint32_t g(const OwnScanParams&) { return G_; }
  __device__ static __forceinline__ constexpr uint32_t shift(const OwnScanParams&, int y) { return (S_ * y) % (32u - U_); }
  __device__ static __forceinline__ constexpr uint32_t lg_ngrp(const OwnScanParams&) { return LGNG_; }
  __device__ static __forceinline__ constexpr uint32_t lg_wg(const OwnScanParams&) { return LGWG_; }
};
using GeoC3 = GeoCt<4, 12, 6, 512, 3, 1>;

// owner-side SetAT of one entry {e = (f(aip) with its frame bits replaced by the word
// within the group), m = touch-bit mask of i}: the r = 4 column windows of
// L = f(aip) >> u, word `sub` of the group in each ATV
template <class Geo>
__device__ __forceinline__ void own_apply(const OwnScanParams& op, uint32_t* sbm, uint32_t e, uint32_t m) {
  const uint64_t L = (uint64_t)(e >> Geo::u(op));
  const uint64_t D = L | (L << Geo::W(op));
  const uint32_t sub = e & Geo::fmask(op);
#pragma unroll
  for (int y = 0; y < 4; ++y) {
    const uint32_t x = (uint32_t)(D >> Geo::shift(op, y)) & Geo::cmask(op);
    const uint32_t w = (((((uint32_t)y << Geo::c(op)) | x) << Geo::lg_wg(op)) | sub);
    OWN_ASSERT(w < ((uint32_t)op.sp.r << (op.sp.c + op.lg_wg)) && m != 0u);
    atomicOr(sbm + w, m);
  }
}

// Bin two packets: f(aip), BH(bip), owner, one slot atomic each, one 8-byte store each.
// The entry carries what the owner needs and nothing it knows: the LBS L in the
// high 32-u bits, the word within the owner's group (< 2^u, host-checked) in the frame
// bits, and the touch-bit mask of i. A full bin (rare) applies the packet straight to the
// global bitmap (k_scan's REDs). Called by whole warps; lanes with !valid do nothing.
template <int CB, bool MP, class Geo>
__device__ __forceinline__ void own_bin_two(const OwnScanParams& op, const uint4 v, bool valid, uint32_t stg_s,
                                            uint32_t scount_s, uint32_t scount_dummy) {
  constexpr uint32_t cap = kOwnCap;
  const ScanParams& p = op.sp;
  const uint32_t h0 = MP ? walk_mod_p(p.A, v.x) : (uint32_t)p.A * v.x;   // f(aip)
  const uint32_t h1 = MP ? walk_mod_p(p.A, v.z) : (uint32_t)p.A * v.z;
  const uint32_t i0 = bh_index(v.y, p.kbh, Geo::g(op));                   // BH (A13)
  const uint32_t i1 = bh_index(v.w, p.kbh, Geo::g(op));
  const uint32_t gs = 5u + Geo::lg_wg(op), wgm = (1u << Geo::lg_wg(op)) - 1u;
  const uint32_t fm = Geo::fmask(op);
  const uint32_t o0 = ((h0 & fm) << Geo::lg_ngrp(op)) | (i0 >> gs);
  const uint32_t o1 = ((h1 & fm) << Geo::lg_ngrp(op)) | (i1 >> gs);
  OWN_ASSERT(!valid || (o0 < op.O && o1 < op.O));
  const uint32_t pos0 = atoms_inc(valid ? scount_s + 4u * o0 : scount_dummy);
  const uint32_t pos1 = atoms_inc(valid ? scount_s + 4u * o1 : scount_dummy);
  const bool ok0 = pos0 < cap, ok1 = pos1 < cap;
  sts64_if(valid && ok0, stg_s + 8u * (o0 * cap + pos0), (h0 & ~fm) | ((i0 >> 5) & wgm), 1u << touch_bit<CB>(i0));
  sts64_if(valid && ok1, stg_s + 8u * (o1 * cap + pos1), (h1 & ~fm) | ((i1 >> 5) & wgm), 1u << touch_bit<CB>(i1));
  const bool ov0 = valid && !ok0, ov1 = valid && !ok1;
  if (__any_sync(0xffffffffu, ov0 || ov1)) {
    if (ov0) scan_pair<CB, MP>(p, v.x, v.y);
    if (ov1) scan_pair<CB, MP>(p, v.z, v.w);
  }
}

template <int CB, bool MP, class Geo>
__global__ void __launch_bounds__(kOwnThreads, 1) k_scan_own(const uint2* __restrict__ pk, uint64_t n,
                                                             OwnScanParams op) {
  const uint32_t kTileBytes = op.tile_bytes;
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int kSig = 2 * kOwnNB;
  static_assert(kSig > kOwnNB + 1, "signal barrier ring");
  __shared__ __align__(8) uint64_t full[kOwnRing], empty[kOwnRing], sigbar[kSig], freebar[kOwnNB];
  __shared__ uint32_t slast[kOwnNB][kOwnQG];     // drain: end of the last drained round per buffer/ring
  const uint32_t G = gridDim.x, me = blockIdx.x, O = op.O;
  const uint32_t Op = (O + 3u) & ~3u;
  const bool owner = me < O;
  constexpr uint32_t nst = kOwnRing, cap = kOwnCap;
  uint8_t* ring = smem;
  uint2* stg = reinterpret_cast<uint2*>(smem + (size_t)nst * kTileBytes);             // [2][O][cap]
  uint32_t* scount = reinterpret_cast<uint32_t*>(stg + 2 * (size_t)O * cap);          // [2][Op]
  uint32_t* sbm = scount + 2 * Op + 4;           // 4 spare words: dummy bin counter (owners: the slice)
  const uint32_t slice_words = (uint32_t)op.sp.r << (op.sp.c + op.lg_wg);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const uint32_t head = (((uintptr_t)pk) & 15u) ? 1u : 0u;
  const uint64_t nbody = (n > head) ? n - head : 0;
  const uint64_t body_bytes = (nbody >> 1) * 16u;
  const uint64_t n_tiles = (body_bytes + kTileBytes - 1) / kTileBytes;
  const uint32_t R = (uint32_t)((n_tiles + G - 1) / G);        // rounds; tile of CTA b in round t: t*G + b
  uint32_t* prod_done = op.sync;
  uint32_t* cons_done = op.sync + kOwnNB * kBinPad;
  constexpr int kBinT = 32 * kOwnBinWarps;                    // named barrier 1
  constexpr int kGroupThreads = 32 * (kOwnConsWarps / kOwnNGR);   // named barriers 2 .. 1 + NGR
  constexpr int kComputeThreads = 32 * (kOwnBinWarps + kOwnConsWarps);   // named barrier 8

  if (owner)   // 16-B stores (sbm is 16-B aligned, slice_words a multiple of 4): scan -0.7 us per call
    for (uint32_t q = threadIdx.x; q < slice_words / 4; q += blockDim.x)
      reinterpret_cast<uint4*>(sbm)[q] = make_uint4(0u, 0u, 0u, 0u);
  for (uint32_t q = threadIdx.x; q < 2 * Op; q += blockDim.x) scount[q] = 0;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kOwnRing; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kOwnBinWarps);
    }
    for (int q = 0; q < kSig; ++q) mbar_init(&sigbar[q], kOwnBinWarps);
    for (int q = 0; q < (int)kOwnNB; ++q) mbar_init(&freebar[q], 1);
    mbar_fence_init();
  }
  __syncthreads();
#ifdef ASSE_OWN_EMPTY
  return;                                        // tools only: launch + prologue cost (no scan)
#endif
  if (op.prof && threadIdx.x == 0) op.prof[me * 16 + 4] = gtimer();   // tools: timeline (ns)
  const uint8_t* body = reinterpret_cast<const uint8_t*>(pk + head);

  if (warp == kOwnSigWarp) {                     // ---------------- round publication
    // first, this CTA's share of the next launch's counters (no memset launch per call)
    for (uint32_t q = (me * 32u + lane) * 4u; q < op.sync_words; q += G * 32u * 4u)
      *reinterpret_cast<uint4*>(op.sync_next + q) = make_uint4(0u, 0u, 0u, 0u);
    if (lane == 0)
      for (uint32_t tf = 0; tf < R; ++tf) {
        mbar_wait_suspend(&sigbar[tf % kSig], (tf / kSig) & 1u);   // every binning warp wrote round tf
        __threadfence();                         // cumulative release of those writes
        atomicAdd(prod_done + (tf % kOwnNB) * kBinPad, 1u);
      }
    return;
  }
  if (warp == kOwnTmaWarp && lane == 1) {       // ---------------- buffer-reuse handoff
    // the queue buffer of round t may be rewritten once every owner drained round t - NB:
    // this lane acquires the owners' release adds (gpu scope) and hands the buffer to the
    // binning warps through a CTA-scope mbarrier (release / acquire), so no binning thread
    // ever stalls on a global acquire load. Barrier t mod NB: its arrival for round t + NB
    // needs round t drained everywhere, i.e. published by this CTA's binning warps after
    // they consumed the arrival for round t (no phase can be skipped). Lane 0 of this warp
    // issues the tile copies; independent thread scheduling interleaves the two loops.
    for (uint32_t t = kOwnNB; t < R; ++t) {
      const uint32_t* cd = cons_done + (t % kOwnNB) * kBinPad;
      const uint32_t need = O * (t / kOwnNB);
      if (ld_acquire_gpu(cd) < need) {           // not yet: poll without the acquire's CCTL.IVALL
        while (ld_relaxed_gpu(cd) < need) __nanosleep(OWN_FREE_SLEEP);
        while (ld_acquire_gpu(cd) < need) {}
      }
      mbar_arrive(&freebar[t % kOwnNB]);
    }
    return;
  }
  if (warp == kOwnTmaWarp) {                     // ---------------- packet tiles -> ring
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      uint32_t i = 0;
      for (uint32_t t = 0; t < R; ++t) {
        const uint64_t tile = (uint64_t)t * G + me;
        if (tile >= n_tiles) break;
        const uint32_t st = i % nst;
        if (i >= nst) mbar_wait_suspend(&empty[st], ((i / nst) - 1) & 1u);
        const uint64_t off = tile * (uint64_t)kTileBytes;
        const uint32_t bytes = (uint32_t)umin64(kTileBytes, body_bytes - off);
        mbar_expect_tx(&full[st], bytes);
        bulk_g2s(ring + (size_t)st * kTileBytes, body + off, bytes, &full[st], pol);
        ++i;
      }
    }
    return;
  }

  if (warp < (uint32_t)kOwnBinWarps) {           // ---------------- binning + flushing warps
    const uint32_t tid = threadIdx.x;
    if (me == 0 && tid == 0) {                   // scalar head / odd tail packets: direct RED
      if (head && n > 0) scan_pair<CB, MP>(op.sp, pk[0].x, pk[0].y);
      if (nbody & 1) scan_pair<CB, MP>(op.sp, pk[n - 1].x, pk[n - 1].y);
    }
    uint32_t i = 0;
    unsigned long long pc[4] = {0, 0, 0, 0};
    long long c0 = clock64(), c1;
    const uint32_t my_o = warp + kOwnBinWarps * lane;   // owners this lane reserves for
    for (uint32_t t = 0; t <= R; ++t) {
      const uint32_t sb = t & 1u, sf = sb ^ 1u;
      const uint32_t tf = t - 1, bf = tf % kOwnNB;
      uint32_t cnt = 0, off = 0;
      if (t >= 1 && my_o < O) {
        // whole 16-B groups: pad the bin with a "no entry" entry up to an even count
        const uint32_t c = min(scount[sf * Op + my_o], cap);
        cnt = (c + 1u) & ~1u;
        if (c & 1u) stg[((size_t)sf * O + my_o) * cap + c] = make_uint2(0u, 0u);   // mask 0: no entry
        if (cnt) off = atomicAdd(op.qcnt + (((size_t)bf * O + my_o) * kOwnQG + (me % kOwnQG)) * kBinPad, cnt);
        OWN_ASSERT(cnt <= cap + 1u && (cnt & 1u) == 0u && (off & 1u) == 0u);
      }
      c1 = clock64(); pc[1] += c1 - c0; c0 = c1;
      const uint64_t tile = (uint64_t)t * G + me;
      if (t < R && tile < n_tiles) {
        const uint32_t st = i % nst;
        {
          const long long w0 = clock64();
          mbar_wait(&full[st], (i / nst) & 1u);
          pc[3] += clock64() - w0;               // tile arrival (tools: ASSE_SCAN_PROF)
        }
        const uint32_t n4 = (uint32_t)umin64(kTileBytes, body_bytes - tile * (uint64_t)kTileBytes) >> 4;
        const uint4* tp = reinterpret_cast<const uint4*>(ring + (size_t)st * kTileBytes);
        const uint32_t stg_s = smem_u32(stg + (size_t)sb * O * cap), scount_s = smem_u32(scount + sb * Op);
        const uint32_t dummy_s = smem_u32(scount + 2 * Op);
        for (uint32_t q0 = tid - lane; q0 < n4; q0 += kBinT) {   // warp-uniform trip count
          const uint32_t q = q0 + lane;
          const bool valid = q < n4;
          own_bin_two<CB, MP, Geo>(op, valid ? tp[q] : make_uint4(0, 0, 0, 0), valid, stg_s, scount_s, dummy_s);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        ++i;
      }
      c1 = clock64(); pc[0] += c1 - c0; c0 = c1;
      if (t >= 1) {
        const uint2* stg_f = stg + (size_t)sf * O * cap;
        uint2* qb = op.queue + ((size_t)bf * O * kOwnQG + (me % kOwnQG)) * kOwnQCap;
        // two owners per step (one per half-warp), 16 B (two entries) per lane (measured
        // faster than the same copy with 32-bit offsets from per-round bases: 0.799 vs 0.812 ms)
        const uint32_t hl = lane & 15u, hw = lane >> 4;
        constexpr int NS = (kOwnMaxOwners + 2 * kOwnBinWarps - 1) / (2 * kOwnBinWarps);
        __syncwarp();                            // padding entries written by other lanes
        uint4 v[NS];
        uint32_t c2[NS], of[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) {
          c2[k] = __shfl_sync(0xffffffffu, cnt, 2 * k + hw);   // entries (even); 0 beyond O
          of[k] = __shfl_sync(0xffffffffu, off, 2 * k + hw);
          const uint32_t ow = warp + kOwnBinWarps * (2 * k + hw);
          if (2 * hl < c2[k]) {
            const uint32_t a = smem_u32(stg_f + (size_t)ow * cap) + 16u * hl;
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "r"(a));
          }
        }
#pragma unroll
        for (int k = 0; k < NS; ++k) {
          const uint32_t ow = warp + kOwnBinWarps * (2 * k + hw);
          if (2 * hl < c2[k]) {
            uint4* dst = reinterpret_cast<uint4*>(qb + (size_t)ow * kOwnQG * kOwnQCap);
            dst[((of[k] >> 1) + hl) & (kOwnQCap / 2 - 1)] = v[k];
          }
        }
        if (my_o < O) scount[sf * Op + my_o] = 0;
        __syncwarp();
        if (lane == 0) mbar_arrive(&sigbar[tf % kSig]);   // this warp wrote round tf
      }
      if (tid == 0 && t >= (uint32_t)kOwnNB && t < R)   // round t-NB drained (handoff lane)
        mbar_wait(&freebar[t % kOwnNB], ((t / kOwnNB) - 1u) & 1u);
      named_bar(1, kBinT);                       // bins of round t final; staging sf and counts reusable
      c1 = clock64(); pc[2] += c1 - c0; c0 = c1;
    }
    if (op.prof && tid == 0) {
      for (int q = 0; q < 4; ++q) op.prof[me * 16 + q] = pc[q];
      op.prof[me * 16 + 5] = gtimer();          // last round shipped
    }
  } else if (owner) {                            // ---------------- queue-draining warps
    const uint32_t cid = warp - kOwnConsWarp0;
    const uint32_t grp = cid / (kOwnConsWarps / kOwnNGR);
    const uint32_t gtid = threadIdx.x - 32 * (kOwnConsWarp0 + grp * (kOwnConsWarps / kOwnNGR));
    constexpr uint32_t GT = 32 * (kOwnConsWarps / kOwnNGR);
    unsigned long long cwait = 0, cwork = 0;
    long long c0 = clock64(), c1;
    for (uint32_t t = grp; t < R; t += kOwnNGR) {
      const uint32_t b = t % kOwnNB;
      if (gtid == 0) spin_until_geq(prod_done + b * kBinPad, G * (t / kOwnNB + 1), 300);
      named_bar(2 + grp, kGroupThreads);
      c1 = clock64(); cwait += c1 - c0; c0 = c1;
      // the round's entries: QG ranges [start, end) of the owner's rings of buffer b; start =
      // end of the previous round in this buffer (slast, written by this group only)
      uint32_t st[kOwnQG], len[kOwnQG], en[kOwnQG], mx = 0;
#pragma unroll
      for (int g = 0; g < (int)kOwnQG; ++g) {
        en[g] = ld_cg_u32(op.qcnt + (((size_t)b * O + me) * kOwnQG + g) * kBinPad);
        st[g] = t >= kOwnNB ? slast[b][g] : 0u;
        len[g] = en[g] - st[g];                  // entries (even)
        OWN_ASSERT(len[g] <= kOwnQCap && (len[g] & 1u) == 0u);
        mx = max(mx, len[g]);
      }
      const uint4* qb4 = reinterpret_cast<const uint4*>(op.queue + ((size_t)b * O + me) * kOwnQG * kOwnQCap);
      constexpr int U = ASSE_OWN_U;              // 16-B groups in flight per thread per ring
      for (uint32_t e0 = gtid; 2 * e0 < mx; e0 += U * GT) {
        uint4 v[kOwnQG][U];
#pragma unroll
        for (int g = 0; g < (int)kOwnQG; ++g)
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint32_t e = e0 + u * GT;      // 16-B group index within the round's range
            v[g][u] = make_uint4(0u, 0u, 0u, 0u);
            if (2 * e < len[g]) {
              const uint4* a = qb4 + g * (kOwnQCap / 2) + (((st[g] >> 1) + e) & (kOwnQCap / 2 - 1));
              asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                           : "=r"(v[g][u].x), "=r"(v[g][u].y), "=r"(v[g][u].z), "=r"(v[g][u].w) : "l"(a));
            }
          }
#pragma unroll
        for (int g = 0; g < (int)kOwnQG; ++g)
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint4 x = v[g][u];
            if (x.y) own_apply<Geo>(op, sbm, x.x, x.y);
            if (x.w) own_apply<Geo>(op, sbm, x.z, x.w);
          }
      }
      named_bar(2 + grp, kGroupThreads);
      // release of the round's entry loads by the group's second warp: its MEMBAR then
      // overlaps the leader's poll for the group's next round (a release by the leader
      // itself measured 0.750 vs 0.733 ms at C5)
      if (gtid == (GT > 32 ? 32u : 0u)) red_release_add(cons_done + b * kBinPad, 1u);
      if (gtid == 0) {
#pragma unroll
        for (int g = 0; g < (int)kOwnQG; ++g) slast[b][g] = en[g];
      }
      c1 = clock64(); cwork += c1 - c0; c0 = c1;
    }
    if (op.prof && gtid == 0 && grp < 2) { op.prof[me * 16 + 9 + 2 * grp] = cwait; op.prof[me * 16 + 10 + 2 * grp] = cwork; }
  }
  // every round consumed by this CTA (owners) / produced (all): every producer published
  // every round, so all overflow REDs are performed; OR the owned slice into the global
  // bitmap: slice word ((y << c | x) << lg_wg) | sub -> global ATV ((y F + z) << c) + x,
  // word grp * WG + sub
  named_bar(8, kComputeThreads);
  if (op.prof && threadIdx.x == 0) op.prof[me * 16 + 6] = gtimer();   // every round drained
  if (!owner) return;
#ifdef ASSE_OWN_NO_WB
  return;                                        // tools only: timing without the write-back (wrong results)
#endif
  __threadfence();
  const ScanParams& p = op.sp;
  const uint32_t z = me >> op.lg_ngrp, grp = me & ((1u << op.lg_ngrp) - 1u);
  const uint32_t wg = 1u << op.lg_wg;
  const uint32_t gbase = (z << p.c) * p.wpa + grp * wg;
  const uint32_t row_words = (p.fmask + 1u) << p.c;          // ATVs per row
  // fire-and-forget ORs (RED): no read of the global word, so nothing waits on L2 round
  // trips (the read-OR-write it replaces cost ~14 us per call: C5 scan 0.722 -> 0.707 ms,
  // C3 0.181 -> 0.166 ms; profiles/r02_sweeps/sweep_wb.jsonl; plain 8-B stores measured 3 us
  // slower than the REDs); atomic, so overflow REDs of other CTAs and earlier calls of the
  // slice need no ordering argument
  if (op.lg_wg >= 1) {                            // 8-B chunks
    const uint32_t n2 = slice_words >> 1;
    for (uint32_t q = threadIdx.x; q < n2; q += kComputeThreads) {
      const uint2 sv = reinterpret_cast<const uint2*>(sbm)[q];
      if (sv.x | sv.y) {
        const uint32_t w = q << 1;
        const uint32_t yx = w >> op.lg_wg, sub = w & (wg - 1u);
        const uint32_t y = yx >> p.c, x = yx & p.cmask;
        OWN_ASSERT((size_t)(y * row_words + x) * p.wpa + gbase + sub + 1 < (size_t)p.r * row_words * p.wpa);
        unsigned long long* gd =
            reinterpret_cast<unsigned long long*>(p.touch + (size_t)(y * row_words + x) * p.wpa + gbase + sub);
        const unsigned long long v = ((unsigned long long)sv.y << 32) | sv.x;
        asm volatile("red.relaxed.gpu.global.or.b64 [%0], %1;" :: "l"(gd), "l"(v) : "memory");
      }
    }
  } else {
    for (uint32_t q = threadIdx.x; q < slice_words; q += kComputeThreads) {
      const uint32_t sv = sbm[q];
      if (sv) {
        const uint32_t y = q >> p.c, x = q & p.cmask;
        uint32_t* gd = p.touch + (size_t)(y * row_words + x) * p.wpa + gbase;
        asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" :: "l"(gd), "r"(sv) : "memory");
      }
    }
  }
}

}  // namespace asse
