// asse_scan_bin.cuh — Alg. 3 with the touch bitmap held in shared memory.
//
// Why: k_scan issues r random 4-byte RED.OR per packet into the L2-resident touch
// bitmap and runs at ~0.9 of the measured random-op ceiling (~188 Gop/s, 1.56
// SM-cycles per update, tools/l2bench.cu). A random shared-memory atomic costs 0.18
// SM-cycles and a coalesced 16-byte global access a small fraction of that
// (tools/smembench.cu, profiles/r01_smembench.txt). The bitmaps of the BASELINE
// geometries (16 MiB at C3-C5) fit in the sum of the SMs' shared memories, so
// (DESIGN.md §5.4):
//
//  * one persistent CTA per SM (cooperative launch: all CTAs co-resident); CTA o OWNS
//    words [o*wpo, (o+1)*wpo) of the binned rows and keeps them in shared memory for the
//    whole call; rows y < RR keep k_scan's RED route into L2 (RR = 1 at C3-C5);
//  * round t: every CTA takes one packet tile (2048 packets at RR = 1, TMA bulk copy into
//    a 2-stage ring); 16 binning warps compute the SetAT targets exactly as k_scan does and
//    bin the binned rows' updates by owner in a double-buffered staging area (one shared
//    atomic for the slot + a predicated store);
//  * while round t is binned, round t-1's bins are padded to 16 B, their ranges reserved in
//    the owner rings [t mod NB][o][producer group] with one global atomicAdd each (issued
//    before the binning, so its latency hides) and copied with 16-byte stores; a signal
//    warp publishes the round (release fence + counter);
//  * eight draining warps (two groups, round parity) wait for a round to be published by
//    every CTA and apply their owner's entries with shared-memory atomicOr;
//  * at the end every CTA ORs its owned words into the global touch bitmap.
//
// A bin that overflows its CAP entries in one round falls back to a direct RED.OR of
// the update into the global bitmap (same result: the write-back ORs). The state after
// the call is bit-identical to k_scan's: the set of touch bits is a union, independent
// of order (SetAT is idempotent within a slice).
#pragma once
#include "asse_kernels.cuh"

namespace asse {

constexpr int kBinBinWarps = 16;                           // binning + shipping warps
constexpr int kBinConsWarps = 8;                           // queue-draining warps, two groups (round parity)
constexpr int kBinConsWarp0 = kBinBinWarps;
constexpr int kBinTmaWarp = kBinConsWarp0 + kBinConsWarps; // packet tiles -> shared ring (TMA)
constexpr int kBinSigWarp = kBinTmaWarp + 1;               // publishes rounds (release fence off the
                                                           // binning warps' path)
constexpr int kBinThreads = 32 * (kBinSigWarp + 1);
constexpr int kBinRing = 2;                                // packet-tile ring stages
constexpr int kBinCap = 88;                                // staged entries per (owner, round) in a CTA
constexpr int kBinStride = 92;                             // words between bins: bin o starts at bank
                                                           // 4o mod 32, so equal slots of different bins
                                                           // do not collide (16-B aligned)
constexpr int kBinNB = 4;                                  // queue buffers (rounds) in flight
constexpr uint32_t kBinQG = 4;                             // producer groups (CTA index mod 4) with separate
                                                           // queues: 4x fewer reservations per counter
constexpr uint32_t kBinQCap = 4096;                        // ring words per (buffer, owner, group)
                                                           // >= ceil(G / QG) * kBinCap
constexpr uint32_t kBinPad = 64;                           // words between counters: one 256-B L2 line
                                                           // pair (one L2 slice) per counter
constexpr uint32_t kBinMinTilesPerCta = 8;                 // below: k_scan is used
constexpr uint32_t kMaxOwners = 160;                       // owners (SMs) the kernel is built for

struct BinScanParams {
  ScanParams sp;          // hashing parameters and the global touch bitmap
  uint32_t* queue;        // [NB][G owners][QG][QCAP] rings of entries (local word << 5 | bit)
  uint32_t* qcnt;         // [NB][G owners][QG] x kBinPad: entries ever reserved (monotone per launch)
  uint32_t* sync;         // [2 NB] x kBinPad: rounds published per buffer, then rounds drained; zeroed
                          // per launch
  uint64_t total_words;   // binned words: rows RR..r-1 of the touch bitmap
  uint32_t base_word;     // first binned word (RR rows x 2^(u+c) ATVs x g/32 words)
  uint32_t tile_bytes;    // packets per CTA per round x 8 (4096 binned updates per round)
  uint32_t inv;           // ceil(2^40 / wpo) (< 2^32 for wpo > 256): owner = (w * inv) >> 40, exact for
                          // w < 2^25 (the error term w * (inv - 2^40/wpo) / 2^40 < 1/wpo)
  uint32_t wpo;           // touch words per owner (multiple of 4)
  unsigned long long* prof;  // optional per-CTA phase cycle counters [G][16] (tools; may be null)
};

__host__ __device__ constexpr size_t bin_smem_bytes(uint32_t G, uint32_t wpo, uint32_t tile_bytes) {
  return (size_t)kBinRing * tile_bytes + 2 * (size_t)G * kBinStride * 4 + 2 * (((size_t)G * 4 + 15) & ~(size_t)15) +
         16 + (size_t)wpo * 4;
}

__device__ __forceinline__ uint32_t ld_cg_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Release-add on a monotone counter: every memory access of this thread (and, through the
// preceding bar.sync, of its group) is ordered before the increment (PTX memory model).
#ifndef ASSE_REL_MODE
#define ASSE_REL_MODE 0
#endif
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
#if ASSE_REL_MODE == 0
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
#else   // tools only: the round-1 relaxed add (no release; measurement of the fence's cost)
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
#endif
}
// Poll a monotone counter with acquire loads. The queue protocol's ordering chain (PTX
// memory model, gpu scope):
//   producer: queue stores / overflow REDs -> mbarrier arrive -> signal warp's wait
//             -> fence (__threadfence, cumulative) -> atomicAdd(prod_done)
//   owner:    acquire poll of prod_done -> bar.sync -> .cg loads of the entries; the final
//             write-back of the owned slice follows the acquire of every round's count
//   owner:    entry loads -> bar.sync -> red.release add(cons_done)
//   producer: acquire poll of cons_done -> bar.sync -> stores into the reused ring range
#ifndef ASSE_ACQ_MODE
#define ASSE_ACQ_MODE 0
#endif
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// How a wait acquires (k_scan_own at C5 on B200, tools/sweep.py r02c/r02d; round 1's
// relaxed polls without any acquire: 0.712 ms):
//  0 (default): every poll is an acquire load (LDG.STRONG + CCTL.IVALL): 0.760 ms with the
//     binning warps' own early probe; the acquire reads a value >= target, i.e. the
//     writer's release (fence + atomic add) or a later add of the same counter, so it
//     synchronises with every round it counts
//  1: relaxed polls, then fence.acq_rel.gpu (MEMBAR.SC per wait): 0.870 ms
//  2: relaxed polls, then one acquire load once the target is seen: 0.827 ms (one more
//     serial L2 round trip per wait)
// k_scan_own keeps every global acquire off its binning warps (signal-warp handoff).
__device__ __forceinline__ uint32_t ld_probe_gpu(const uint32_t* p) {
#if ASSE_ACQ_MODE == 0
  return ld_acquire_gpu(p);
#else
  return ld_relaxed_gpu(p);
#endif
}
__device__ __forceinline__ void spin_until_geq(const uint32_t* p, uint32_t target, uint32_t ns = 128) {
#if ASSE_ACQ_MODE == 0
  while (ld_acquire_gpu(p) < target) __nanosleep(ns);   // polls must not steal issue slots
#elif ASSE_ACQ_MODE == 1
  while (ld_relaxed_gpu(p) < target) __nanosleep(ns);
  fence_acq_rel_gpu();
#elif ASSE_ACQ_MODE == 2
  while (ld_relaxed_gpu(p) < target) __nanosleep(ns);
  while (ld_acquire_gpu(p) < target) {}                  // returns at once (monotone counter)
#elif ASSE_ACQ_MODE == 4
  if (ld_acquire_gpu(p) >= target) return;              // ready: one acquire load
  while (ld_relaxed_gpu(p) < target) __nanosleep(ns);   // waiting: polls without CCTL.IVALL
  while (ld_acquire_gpu(p) < target) {}
#else   // 3, tools only: the round-1 relaxed polls without acquire (measures the ordering's cost)
  while (ld_relaxed_gpu(p) < target) __nanosleep(ns);
#endif
}
// after an early probe `seen` of *p: wait until *p >= target with acquire semantics
__device__ __forceinline__ void wait_seen(uint32_t seen, const uint32_t* p, uint32_t target, uint32_t ns = 128) {
  if (seen < target) spin_until_geq(p, target, ns);
#if ASSE_ACQ_MODE == 1
  else fence_acq_rel_gpu();
#elif ASSE_ACQ_MODE == 2
  else spin_until_geq(p, target, ns);                    // one acquire load
#endif
}
// mbarrier wait for warps off the critical path (sleeps between probes)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t phase, uint32_t ns) {
  uint32_t done = 0;
  while (true) {
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done) : "r"(smem_u32(bar)), "r"(phase) : "memory");
    if (done) break;
    __nanosleep(ns);
  }
}
__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(threads) : "memory");
}

// shared-space (32-bit address) accessors: no generic-to-shared conversion per access
__device__ __forceinline__ uint32_t atoms_inc(uint32_t addr) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(addr) : "memory");
  return old;
}
__device__ __forceinline__ void sts_if(bool pred, uint32_t addr, uint32_t v) {
  asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %0, 0;\n @p st.shared.u32 [%1], %2;\n}"
               :: "r"((uint32_t)pred), "r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void red_or_if(bool pred, uint32_t* gaddr, uint32_t v) {
  asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %0, 0;\n @p red.global.or.b32 [%1], %2;\n}"
               :: "r"((uint32_t)pred), "l"(gaddr), "r"(v) : "memory");
}

// The 4 SetAT targets (touch words) of one packet (identical arithmetic to scan_pair;
// the binned kernel serves r = 4, the rows of every BASELINE geometry).
template <int CB, bool MP>
__device__ __forceinline__ void targets4(const ScanParams& p, uint32_t aip, uint32_t bip, uint32_t* w,
                                         uint32_t& tb) {
  const uint32_t h = MP ? walk_mod_p(p.A, aip) : (uint32_t)p.A * aip;   // f(aip)
  const uint32_t z = h & p.fmask;                                         // Z
  const uint64_t L = (uint64_t)(h >> p.u);                                // LBS
  const uint64_t D = L | (L << p.W);                                      // wrap-around
  const uint32_t i = bh_index(bip, p.kbh, p.g);                           // BH (A13)
  const uint32_t wofs = i >> 5;
  tb = touch_bit<CB>(i);
  const uint32_t yz0 = z << p.c;
#pragma unroll
  for (int y = 0; y < 4; ++y) {
    const uint32_t x = (uint32_t)(D >> p.shift[y]) & p.cmask;
    const uint32_t atv = ((uint32_t)y << (p.u + p.c)) + yz0 + x;
    w[y] = atv * p.wpa + wofs;
  }
}

// Bin the 8 updates of two packets: 8 independent shared atomics for the bin slots, then
// predicated stores. A full bin (rare) sends its update straight to the global bitmap.
// Rows y < RR of both packets go straight to the global bitmap (RED.OR into L2, k_scan's
// route); rows y >= RR are binned: RR balances the L2 random-op path against the SMs'
// binning work. Called by whole warps (the overflow vote is warp-wide); lanes with !valid
// do nothing.
template <int CB, bool MP, int RR>
__device__ __forceinline__ void bin_two(const BinScanParams& bp, const uint4 v, bool valid, uint32_t stg_s,
                                        uint32_t scount_s, uint32_t scount_dummy) {
  uint32_t w[8], tb0, tb1;
  targets4<CB, MP>(bp.sp, v.x, v.y, w, tb0);
  targets4<CB, MP>(bp.sp, v.z, v.w, w + 4, tb1);
  constexpr int NB2 = 4 - RR;                    // binned updates per packet
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if ((k & 3) < RR) red_or_if(valid, bp.sp.touch + w[k], 1u << (k < 4 ? tb0 : tb1));
  uint32_t o[2 * NB2], pos[2 * NB2], wl[2 * NB2];
#pragma unroll
  for (int m = 0; m < 2 * NB2; ++m) {
    const int k = (m / NB2) * 4 + RR + (m % NB2);
    wl[m] = w[k] - bp.base_word;
    o[m] = (uint32_t)(((uint64_t)wl[m] * bp.inv) >> 40);   // one IMAD.WIDE
  }
  // lanes without a packet count into a spare counter (index G) instead of branching
#pragma unroll
  for (int m = 0; m < 2 * NB2; ++m) pos[m] = atoms_inc(valid ? scount_s + 4u * o[m] : scount_dummy);
  uint32_t ovf = 0;
#pragma unroll
  for (int m = 0; m < 2 * NB2; ++m) {
    const uint32_t tb = m < NB2 ? tb0 : tb1;
    const uint32_t e = ((wl[m] - o[m] * bp.wpo) << 5) | tb;
    const bool ok = pos[m] < (uint32_t)kBinCap;
    sts_if(valid && ok, stg_s + 4u * (o[m] * kBinStride + pos[m]), e);
    ovf |= (valid && !ok ? 1u : 0u) << m;
  }
  if (__any_sync(0xffffffffu, ovf != 0)) {
#pragma unroll
    for (int m = 0; m < 2 * NB2; ++m)
      if (ovf & (1u << m)) atomicOr(bp.sp.touch + bp.base_word + wl[m], 1u << (m < NB2 ? tb0 : tb1));
  }
}

template <int CB, bool MP, int RR>
__global__ void __launch_bounds__(kBinThreads, 1) k_scan_bin(const uint2* __restrict__ pk, uint64_t n,
                                                             BinScanParams bp) {
  const uint32_t kBinTileBytes = bp.tile_bytes;
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int kSig = 8;
  static_assert(kSig > kBinNB + 1, "signal barrier ring");
  __shared__ __align__(8) uint64_t full[kBinRing], empty[kBinRing], sigbar[kSig];
  const uint32_t G = gridDim.x, me = blockIdx.x;
  const uint32_t Gp = (G + 3u) & ~3u;
  uint8_t* ring = smem;
  uint32_t* stg = reinterpret_cast<uint32_t*>(smem + (size_t)kBinRing * kBinTileBytes);  // [2][G][STRIDE]
  uint32_t* scount = stg + 2 * (size_t)G * kBinStride;                                   // [2][Gp]
  uint32_t* sbm = scount + 2 * Gp + 4;           // 4 spare words: dummy bin counter
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const uint32_t head = (((uintptr_t)pk) & 15u) ? 1u : 0u;
  const uint64_t nbody = (n > head) ? n - head : 0;
  const uint64_t body_bytes = (nbody >> 1) * 16u;
  const uint64_t n_tiles = (body_bytes + kBinTileBytes - 1) / kBinTileBytes;
  const uint32_t R = (uint32_t)((n_tiles + G - 1) / G);        // rounds; tile of CTA b in round t: t*G + b
  uint32_t* prod_done = bp.sync;                 // counter of buffer b at b * kBinPad
  uint32_t* cons_done = bp.sync + kBinNB * kBinPad;
  constexpr int kBinT = 32 * kBinBinWarps;                    // named barrier 1
  constexpr int kGroupThreads = 32 * (kBinConsWarps / 2);     // named barriers 2, 3
  constexpr int kComputeThreads = 32 * (kBinBinWarps + kBinConsWarps);   // named barrier 4

  for (uint32_t q = threadIdx.x; q < bp.wpo; q += blockDim.x) sbm[q] = 0;
  for (uint32_t q = threadIdx.x; q < 2 * Gp; q += blockDim.x) scount[q] = 0;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kBinRing; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kBinBinWarps);
    }
    for (int q = 0; q < kSig; ++q) mbar_init(&sigbar[q], kBinBinWarps);
    mbar_fence_init();
  }
  __syncthreads();
  const uint8_t* body = reinterpret_cast<const uint8_t*>(pk + head);

  if (warp == kBinSigWarp) {                     // ---------------- round publication
    // the binning warps run at most NB + 1 rounds ahead of this warp (they wait for rounds
    // NB back to be drained, which needs them published), so kSig > NB + 1 barriers suffice
    for (uint32_t tf = 0; tf < R; ++tf) {
      mbar_wait_sleep(&sigbar[tf % kSig], (tf / kSig) & 1u, 400);   // every binning warp wrote round tf
      if (lane == 0) {
        __threadfence();                         // cumulative release of those writes
        atomicAdd(prod_done + (tf % kBinNB) * kBinPad, 1u);
      }
      __syncwarp();
    }
    return;
  }
  if (warp == kBinTmaWarp) {                     // ---------------- packet tiles -> ring
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      uint32_t i = 0;
      for (uint32_t t = 0; t < R; ++t) {
        const uint64_t tile = (uint64_t)t * G + me;
        if (tile >= n_tiles) break;
        const uint32_t st = i % kBinRing;
        if (i >= (uint32_t)kBinRing) mbar_wait_sleep(&empty[st], ((i / kBinRing) - 1) & 1u, 1000);
        const uint64_t off = tile * (uint64_t)kBinTileBytes;
        const uint32_t bytes = (uint32_t)umin64(kBinTileBytes, body_bytes - off);
        mbar_expect_tx(&full[st], bytes);
        bulk_g2s(ring + (size_t)st * kBinTileBytes, body + off, bytes, &full[st], pol);
        ++i;
      }
    }
    return;
  }

  if (warp < (uint32_t)kBinBinWarps) {           // ---------------- binning + flushing warps
    const uint32_t tid = threadIdx.x;
    if (me == 0 && tid == 0) {                   // scalar head / odd tail packets: direct RED
      if (head && n > 0) scan_pair<CB, MP>(bp.sp, pk[0].x, pk[0].y);
      if (nbody & 1) scan_pair<CB, MP>(bp.sp, pk[n - 1].x, pk[n - 1].y);
    }
    uint32_t i = 0;
    unsigned long long pc[3] = {0, 0, 0};
    long long c0 = clock64(), c1;
    // iteration t: reserve queue space for round t-1 (staging (t-1)&1), bin round t into
    // staging t&1 (hiding the reservation latency), copy round t-1 into the reserved ranges.
    // Owners of this warp: o = warp + kBinBinWarps * l for lanes l with o < G.
    const uint32_t my_o = warp + kBinBinWarps * lane;
    for (uint32_t t = 0; t <= R; ++t) {
      const uint32_t sb = t & 1u, sf = sb ^ 1u;
      const uint32_t tf = t - 1, bf = tf % kBinNB;
      uint32_t cnt = 0, off = 0;
      // the end-of-iteration barrier (below) made staging sf final and queue buffer bf free
      if (t >= 1) {
        if (my_o < G) {
          // whole 16-B groups: pad the bin with "no entry" words up to a multiple of 4
          const uint32_t c = min(scount[sf * Gp + my_o], (uint32_t)kBinCap);
          cnt = (c + 3u) & ~3u;
          uint32_t* bin = stg + ((size_t)sf * G + my_o) * kBinStride;
          for (uint32_t q = c; q < cnt; ++q) bin[q] = 0xFFFFFFFFu;
          if (cnt) off = atomicAdd(bp.qcnt + (((size_t)bf * G + my_o) * kBinQG + (me % kBinQG)) * kBinPad, cnt);
        }
      }
      c1 = clock64(); pc[1] += c1 - c0; c0 = c1;
      // the drain count the next reservation (round t into buffer t % NB) waits for, loaded
      // early so its latency hides behind the binning
      uint32_t seen = 0;
      const uint32_t need = G * (t / kBinNB);
      if (tid == 0 && t >= (uint32_t)kBinNB && t < R) seen = ld_probe_gpu(cons_done + (t % kBinNB) * kBinPad);
      if (t < R) {
        const uint64_t tile = (uint64_t)t * G + me;
        if (tile < n_tiles) {
          const uint32_t st = i % kBinRing;
          mbar_wait(&full[st], (i / kBinRing) & 1u);
          const uint32_t n4 = (uint32_t)umin64(kBinTileBytes, body_bytes - tile * (uint64_t)kBinTileBytes) >> 4;
          const uint4* tp = reinterpret_cast<const uint4*>(ring + (size_t)st * kBinTileBytes);
          const uint32_t stg_s = smem_u32(stg + (size_t)sb * G * kBinStride), scount_s = smem_u32(scount + sb * Gp);
          for (uint32_t q0 = tid - lane; q0 < n4; q0 += kBinT) {   // warp-uniform trip count
            const uint32_t q = q0 + lane;
            const bool valid = q < n4;
            bin_two<CB, MP, RR>(bp, valid ? tp[q] : make_uint4(0, 0, 0, 0), valid, stg_s, scount_s,
                            smem_u32(scount + 2 * Gp));
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[st]);
          ++i;
        }
      }
      c1 = clock64(); pc[0] += c1 - c0; c0 = c1;
      if (t >= 1) {
        const uint32_t* stg_f = stg + (size_t)sf * G * kBinStride;
        uint32_t* qb = bp.queue + ((size_t)bf * G * kBinQG + (me % kBinQG)) * kBinQCap;
        // two owners per step (one per half-warp), 16 B per lane: staged bin -> ring; all
        // shared loads of the warp's owners are issued before the global stores
        const uint32_t hl = lane & 15u, hw = lane >> 4;
        const uint32_t src_s = smem_u32(stg_f + (size_t)(warp + kBinBinWarps * hw) * kBinStride) + 16u * hl;
        uint4* dst = reinterpret_cast<uint4*>(qb + (size_t)(warp + kBinBinWarps * hw) * kBinQG * kBinQCap);
        constexpr uint32_t kSrcStep = 2 * kBinBinWarps * kBinStride * 4;    // bytes between steps
        constexpr size_t kDstStep = 2 * (size_t)kBinBinWarps * kBinQG * kBinQCap / 4;
        constexpr int NS = (kMaxOwners + 2 * kBinBinWarps - 1) / (2 * kBinBinWarps);   // steps
        uint4 v[NS];
        uint32_t c4[NS], of[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) {
          c4[k] = __shfl_sync(0xffffffffu, cnt, 2 * k + hw);   // 0 beyond nown
          of[k] = __shfl_sync(0xffffffffu, off, 2 * k + hw);
          const uint32_t a = src_s + k * kSrcStep;
          if (4 * hl < c4[k])
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "r"(a));
        }
#pragma unroll
        for (int k = 0; k < NS; ++k)
          if (4 * hl < c4[k]) dst[k * kDstStep + (((of[k] >> 2) + hl) & (kBinQCap / 4 - 1))] = v[k];
        // bins longer than 64 entries: 16-B groups 16.. of those owners (rare)
        if (kBinCap > 64) {
#pragma unroll
          for (int k = 0; k < NS; ++k)
            if (4 * (hl + 16) < c4[k]) {
              uint4 x;
              asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                           : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w) : "r"(src_s + k * kSrcStep + 256u));
              dst[k * kDstStep + (((of[k] >> 2) + hl + 16) & (kBinQCap / 4 - 1))] = x;
            }
        }
        if (my_o < G) scount[sf * Gp + my_o] = 0;
        __syncwarp();
        if (lane == 0) mbar_arrive(&sigbar[tf % kSig]);   // this warp wrote round tf (release.cta)
      }
      if (tid == 0 && t >= (uint32_t)kBinNB && t < R)
        wait_seen(seen, cons_done + (t % kBinNB) * kBinPad, need);   // round t-NB drained everywhere
      named_bar(1, kBinT);                       // bins of round t final; staging sf and counts reusable
      c1 = clock64(); pc[2] += c1 - c0; c0 = c1;
    }
    if (bp.prof && tid == 0)
      for (int q = 0; q < 3; ++q) bp.prof[me * 16 + q] = pc[q];
  } else {                                       // ---------------- queue-draining warps
    const uint32_t cid = warp - kBinConsWarp0;
    const uint32_t grp = cid / (kBinConsWarps / 2);
    const uint32_t gtid = threadIdx.x - 32 * (kBinConsWarp0 + grp * (kBinConsWarps / 2));
    constexpr uint32_t GT = 32 * (kBinConsWarps / 2);
    uint32_t last[2][kBinQG];                    // this group's buffers b = grp and grp + 2
#pragma unroll
    for (int g = 0; g < (int)kBinQG; ++g) last[0][g] = last[1][g] = 0;
    unsigned long long cwait = 0, cwork = 0;
    long long c0 = clock64(), c1;
    for (uint32_t t = grp; t < R; t += 2) {
      const uint32_t b = t % kBinNB, li = (t >> 1) & 1u;
      if (gtid == 0) spin_until_geq(prod_done + b * kBinPad, G * (t / kBinNB + 1), 300);
      named_bar(2 + grp, kGroupThreads);
      c1 = clock64(); cwait += c1 - c0; c0 = c1;
      // the round's entries: QG ranges [last, end) of the owner's rings, drained as one list
      uint32_t st[kBinQG], pre[kBinQG + 1];
      pre[0] = 0;
#pragma unroll
      for (int g = 0; g < (int)kBinQG; ++g) {
        const uint32_t end = ld_cg_u32(bp.qcnt + (((size_t)b * G + me) * kBinQG + g) * kBinPad);
        const uint32_t s0 = li ? last[1][g] : last[0][g];
        st[g] = s0;
        pre[g + 1] = pre[g] + (end - s0);
        if (li) last[1][g] = end; else last[0][g] = end;
      }
      const uint32_t* qb = bp.queue + ((size_t)b * G + me) * kBinQG * kBinQCap;
      uint32_t len[kBinQG], mx = 0;
#pragma unroll
      for (int g = 0; g < (int)kBinQG; ++g) { len[g] = pre[g + 1] - pre[g]; mx = max(mx, len[g]); }
      constexpr int U = 2;                       // 16-B groups in flight per thread per ring
      const uint4* qb4 = reinterpret_cast<const uint4*>(qb);
      for (uint32_t e0 = gtid; 4 * e0 < mx; e0 += U * GT) {
        uint4 v[kBinQG][U];
#pragma unroll
        for (int g = 0; g < (int)kBinQG; ++g)
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint32_t e = e0 + u * GT;      // 16-B group index within the round's range
            v[g][u] = make_uint4(~0u, ~0u, ~0u, ~0u);
            if (4 * e < len[g]) {
              const uint4* a = qb4 + g * (kBinQCap / 4) + (((st[g] >> 2) + e) & (kBinQCap / 4 - 1));
              asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                           : "=r"(v[g][u].x), "=r"(v[g][u].y), "=r"(v[g][u].z), "=r"(v[g][u].w) : "l"(a));
            }
          }
#pragma unroll
        for (int g = 0; g < (int)kBinQG; ++g)
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint4 x = v[g][u];
            if (x.x != ~0u) atomicOr(sbm + (x.x >> 5), 1u << (x.x & 31u));
            if (x.y != ~0u) atomicOr(sbm + (x.y >> 5), 1u << (x.y & 31u));
            if (x.z != ~0u) atomicOr(sbm + (x.z >> 5), 1u << (x.z & 31u));
            if (x.w != ~0u) atomicOr(sbm + (x.w >> 5), 1u << (x.w & 31u));
          }
      }
      named_bar(2 + grp, kGroupThreads);
      if (gtid == 0) red_release_add(cons_done + b * kBinPad, 1u);   // entries consumed (values used) before
      c1 = clock64(); cwork += c1 - c0; c0 = c1;
    }
    if (bp.prof && gtid == 0) { bp.prof[me * 16 + 9 + 2 * grp] = cwait; bp.prof[me * 16 + 10 + 2 * grp] = cwork; }
  }
  // every round consumed by this CTA: every producer has published every round, so all
  // overflow REDs are performed; OR the owned words into the global bitmap with one bulk
  // reduction (TMA cp.reduce.async.bulk .or: the owned words are contiguous in global
  // memory), performed in L2 — no read of the global words by the SM
  fence_proxy_async_smem();                     // this thread's shared atomics -> async proxy
  named_bar(4, kComputeThreads);
  const uint64_t w0 = (uint64_t)me * bp.wpo;
  if (threadIdx.x == 0 && w0 < bp.total_words) {
    const uint32_t nw = (uint32_t)umin64(bp.wpo, bp.total_words - w0);   // multiple of 4 (16 B)
    uint32_t* gdst = bp.sp.touch + bp.base_word + w0;
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.or.b32 [%0], [%1], %2;"
                 :: "l"(gdst), "r"(smem_u32(sbm)), "r"(nw * 4u) : "memory");
    bulk_commit();
    bulk_wait0();                                // complete before the CTA's shared memory goes away
  }
}

}  // namespace asse
