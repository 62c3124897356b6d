// asse_kernels.cuh — sm_100a kernels of the ASSE hot path (arXiv 1807.01527).
//
// P:n = PAPER.md line n; A<n> = reading n of DESIGN.md §2. No tensor cores: nothing
// here is a dense contraction. Layout:
//   pool    : AT codes [y][z][x][i], CT = uint8_t (2k <= 126) or uint16_t   (A2)
//   touch   : per-slice SetAT record, g bits per ATV, same [y][z][x] order;
//             bit of AT i inside word i>>5 permuted (touch_bit) for a PRMT fold
//   active  : checkAT(k') result of the last end_slice, g bits per ATV
// The value SetAT writes into AT i during slice t is fully determined by i and t
// (block ACT (C0 + blk(i)) mod 2k), so the scan only records WHICH ATs were
// set (1 bit each, L2-resident) and k_fold writes the codes once per slice.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>


#include "asse_tma.cuh"

namespace asse {

constexpr int kMaxR = 8;       // rows supported by the device path
constexpr int kMaxWorld = 16;  // ranks supported by the peer merge

// ------------------------------------------------------------------ helpers

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ __forceinline__ uint32_t bh_index(uint32_t bip, uint64_t kbh, uint32_t g) {
  // BH (A13): SplitMix64 finalizer of bip ^ K_bh, multiply-shift to [0, g):
  //   z = bip ^ K; z = (z ^ z>>30) * C1; z = (z ^ z>>27) * C2; z ^= z>>31; i = ((z>>32) * g) >> 32
  // in 32-bit halves: the high half of bip ^ K is K's (a warp-uniform constant, so the
  // compiler hoists everything that depends on it), and only the high half of the last
  // product is needed (bit-identical to the 64-bit form; every pool parity test checks it)
  constexpr uint32_t C1L = 0x1CE4E5B9u, C1H = 0xBF58476Du, C2L = 0x133111EBu, C2H = 0x94D049BBu;
  const uint32_t khi = (uint32_t)(kbh >> 32);
  const uint32_t lo = bip ^ (uint32_t)kbh;
  const uint32_t xl = lo ^ __funnelshift_r(lo, khi, 30);
  const uint32_t xh = khi ^ (khi >> 30);
  const uint32_t yl = xl * C1L;
  const uint32_t yh = __umulhi(xl, C1L) + xl * C1H + xh * C1L;
  const uint32_t wl = yl ^ __funnelshift_r(yl, yh, 27);
  const uint32_t wh = yh ^ (yh >> 27);
  const uint32_t vh = __umulhi(wl, C2L) + wl * C2H + wh * C2L;
  return __umulhi(vh ^ (vh >> 31), g);
}

// Bit position of AT i inside touch word i>>5. Lane l of k_fold owns ATs
// 16l..16l+15 of a 512-AT chunk, i.e. half-word (i>>4)&1 of word i>>5; inside
// that half the order makes a PRMT selector one shift + one mask away.
template <int CB>
__device__ __forceinline__ uint32_t touch_bit(uint32_t i) {
  uint32_t half = ((i >> 4) & 1u) << 4;
  if (CB == 1) return half + 4u * (i & 3u) + ((i >> 2) & 3u);   // code 4q+j -> bit 4j+q
  return half + 8u * (i & 1u) + ((i >> 1) & 7u);                // code 2q+j -> bit 8j+q
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// streaming read-only input (packets): no L1 allocation, evict-first in L2
__device__ __forceinline__ uint4 ld_stream(const uint4* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
  return r;
}
// AT pool streamed once per slice: evict-first so the bitmaps stay L2-resident
__device__ __forceinline__ uint4 ld_pool(const uint4* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ void st_pool(uint4* p, uint4 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol) : "memory");
}

// f(x) = A x mod p, p = 2^32 + 15 (the smallest prime above 2^32), with cycle walking
// back into 32 bits (P:305 literal form). Reduction uses
// 2^32 = -15 and 2^64 = 225 (mod p).
constexpr uint64_t kMangleP = 4294967311ULL;
__host__ __device__ __forceinline__ uint64_t mulmod_p(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  const uint64_t lo = a * b, hi = __umul64hi(a, b);
#else
  const unsigned __int128 v = (unsigned __int128)a * b;
  const uint64_t lo = (uint64_t)v, hi = (uint64_t)(v >> 64);
#endif
  int64_t t = (int64_t)(lo & 0xFFFFFFFFull) + (int64_t)(hi * 225u) - 15 * (int64_t)(lo >> 32)
              + 16 * (int64_t)kMangleP;
  const uint64_t u = (uint64_t)t;
  int64_t t2 = (int64_t)(u & 0xFFFFFFFFull) - 15 * (int64_t)(u >> 32);
  if (t2 < 0) t2 += (int64_t)kMangleP;
  return (uint64_t)t2;
}
__host__ __device__ __forceinline__ uint32_t walk_mod_p(uint64_t key, uint32_t x) {
  uint64_t y = mulmod_p(key, x);
  while (y >> 32) y = mulmod_p(key, y);
  return (uint32_t)y;
}

// ------------------------------------------------------------------- scan

struct ScanParams {
  uint32_t* touch;        // touch bitmap, words_per_atv words per ATV
  uint64_t kbh;           // BH key
  uint64_t A;             // mangling key (A8: odd, mod 2^32; or in [1, p-1] for MP)
  uint32_t g, r, u, c, W; // W = 32 - u
  uint32_t fmask, cmask;
  uint32_t wpa;           // touch words per ATV = g/32
  uint32_t shift[kMaxR];  // (s*y) mod W
};

// Alg. 3 for one pair: RRH(aip) -> r ATVs <x_y, y, z>, i = BH(bip),
// SetAT recorded as touch bit i of each ATV.
template <int CB, bool MP>
__device__ __forceinline__ void scan_pair(const ScanParams& p, uint32_t aip, uint32_t bip) {
  const uint32_t h = MP ? walk_mod_p(p.A, aip) : (uint32_t)p.A * aip;   // f(aip)
  const uint32_t z = h & p.fmask;                      // Z(aip) = RBS(f, u)
  const uint64_t L = (uint64_t)(h >> p.u);             // LBS(f, 32-u)
  const uint64_t D = L | (L << p.W);                   // wrap-around view
  const uint32_t i = bh_index(bip, p.kbh, p.g);
  const uint32_t wofs = i >> 5;
  const uint32_t bit = 1u << touch_bit<CB>(i);
  const uint32_t yz0 = z << p.c;
#pragma unroll
  for (int y = 0; y < kMaxR; ++y) {
    if (y < (int)p.r) {
      uint32_t x = (uint32_t)(D >> p.shift[y]) & p.cmask;
      uint32_t atv = ((uint32_t)y << (p.u + p.c)) + yz0 + x;   // ((y*F + z) << c) | x
      atomicOr(p.touch + (size_t)atv * p.wpa + wofs, bit);    // RED.E.OR (no return)
    }
  }
}

constexpr int kScanConsumerWarps = 8;
constexpr int kScanThreads = 32 * (kScanConsumerWarps + 1);   // + 1 producer warp
constexpr uint32_t kScanTileBytes = 16384;                      // 2048 packets per stage
constexpr int kScanStages = 4;
constexpr size_t kScanSmem = (size_t)kScanStages * kScanTileBytes;

// Alg. 3 over a device packet buffer. The 16-B aligned body is streamed through a
// 4-stage shared-memory ring by bulk copies (TMA, cp.async.bulk; one producer warp),
// tile i of this CTA = body tile blockIdx.x + i*gridDim.x; the 8 consumer warps
// hash the packets and issue r RED.OR per packet into the L2-resident touch bitmap.
template <int CB, bool MP = false>
__global__ void __launch_bounds__(kScanThreads) k_scan(const uint2* __restrict__ pk, uint64_t n,
                                                       ScanParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kScanStages], empty[kScanStages];
  const uint32_t head = (((uintptr_t)pk) & 15u) ? 1u : 0u;
  const uint64_t nbody = (n > head) ? n - head : 0;
  const uint64_t body_bytes = (nbody >> 1) * 16u;
  const uint64_t n_tiles = (body_bytes + kScanTileBytes - 1) / kScanTileBytes;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  if (blockIdx.x == 0 && threadIdx.x == 0) {     // scalar head / odd tail packets
    if (head && n > 0) scan_pair<CB, MP>(p, pk[0].x, pk[0].y);
    if (nbody & 1) scan_pair<CB, MP>(p, pk[n - 1].x, pk[n - 1].y);
  }
  const uint64_t my_tiles =
      (n_tiles > blockIdx.x) ? (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kScanStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kScanConsumerWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const uint8_t* body = reinterpret_cast<const uint8_t*>(pk + head);
  if (warp == kScanConsumerWarps) {              // producer warp
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (uint64_t i = 0; i < my_tiles; ++i) {
        const uint32_t st = (uint32_t)(i % kScanStages);
        if (i >= kScanStages) mbar_wait(&empty[st], (uint32_t)((i / kScanStages) - 1) & 1u);
        const uint64_t off = (blockIdx.x + i * gridDim.x) * (uint64_t)kScanTileBytes;
        const uint32_t bytes = (uint32_t)umin64(kScanTileBytes, body_bytes - off);
        mbar_expect_tx(&full[st], bytes);
        bulk_g2s(smem + (size_t)st * kScanTileBytes, body + off, bytes, &full[st], pol);
      }
    }
    return;
  }
  for (uint64_t i = 0; i < my_tiles; ++i) {
    const uint32_t st = (uint32_t)(i % kScanStages);
    mbar_wait(&full[st], (uint32_t)(i / kScanStages) & 1u);
    const uint64_t off = (blockIdx.x + i * gridDim.x) * (uint64_t)kScanTileBytes;
    const uint32_t n4 = (uint32_t)umin64(kScanTileBytes, body_bytes - off) >> 4;
    const uint4* tp = reinterpret_cast<const uint4*>(smem + (size_t)st * kScanTileBytes);
    for (uint32_t q = threadIdx.x; q < n4; q += 32 * kScanConsumerWarps) {
      const uint4 v = tp[q];
      scan_pair<CB, MP>(p, v.x, v.y);
      scan_pair<CB, MP>(p, v.z, v.w);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
}

// ------------------------------------------------------------------- fold

struct FoldParams {
  void* pool;                 // codes
  const uint32_t* touch_src;  // touch bits to fold (local, or the merged bitmap)
  uint32_t* touch_zero;       // touch bitmap to clear for the next slice
  uint32_t* active;           // out: active bits (same layout family)
  unsigned long long* aat;    // out: AAT[y][z], pre-zeroed
  uint32_t* sa_cnt;           // out: |SA(y,z)|, pre-zeroed
  uint32_t* sa_list;          // out: SA(y,z) columns, E per (y,z)
  uint32_t* sa_bits;          // out: SA(y,z) membership bits, pre-zeroed
  uint32_t* n_super;          // out: total super ATVs
  uint64_t n_chunks;          // pool ATs / 512
  const uint32_t* C0;         // ACT base of block 0 for this slice (device scalar)
  uint32_t g, k, kp, a;       // ATV size, window, k', block size a (A7)
  uint32_t c, w_theta;        // column bits, integer super threshold (A15)
  uint32_t lpa_log2;          // log2(lanes per ATV) = log2(g/16)
};

// Element-wise SWAR constants: CB = 1 -> 4 x 7-bit codes per word (guard bit 7),
// CB = 2 -> 2 x 15-bit codes per word (guard bit 15).
template <int CB> struct Swar;
template <> struct Swar<1> {
  static constexpr int NW = 4;      // words per lane (16 codes)
  static constexpr int EPW = 4;     // elements per word
  static constexpr int EB = 8;      // element bits
  static constexpr uint32_t G = 0x80808080u;
  static constexpr uint32_t EMPTY_LO = 127u;
};
template <> struct Swar<2> {
  static constexpr int NW = 8;
  static constexpr int EPW = 2;
  static constexpr int EB = 16;
  static constexpr uint32_t G = 0x80008000u;
  static constexpr uint32_t EMPTY_LO = 32767u;
};

// v in [lo, hi] per element, result in the guard bits (borrow-free: vx elements have
// the guard bit set and lo <= guard-1; HX = hi | guard, v <= guard - 2).
__device__ __forceinline__ uint32_t in_range(uint32_t vx, uint32_t v, uint32_t LO, uint32_t HX) {
  return (vx - LO) & (HX - v);
}

// One 512-AT chunk per warp and pass; lane l owns ATs 16l..16l+15 (16 B of u8 or
// 32 B of u16 codes). For every AT:
//   SetAT fold  v <- ACT(i) if touched this slice                     (Alg. 3)
//   checkAT     active <=> v != 2k and (ACT(i) - v) mod 2k <= k'-1    (Alg. 1)
//   weight      |ATV|^{k'} = popcount over the ATV; AAT
//   super       w >= W_theta -> SA(y,z)
//   preserveAT  for slice t+1 on ATs whose block ACT becomes 0 or k  (Alg. 2)
// The per-AT constants depend only on the AT index, so each lane computes them
// once per launch and keeps them in registers (blocked warp -> chunk mapping).
constexpr int kFoldConsumerWarps = 8;
constexpr int kFoldThreads = 32 * (kFoldConsumerWarps + 1);   // + 1 producer warp
constexpr uint32_t kFoldChunksPerTile = 16;                    // 16 x 512 ATs per stage
constexpr int kFoldStages = 4;   // 6 / 8 stages (2 or 4 out stages): same at u8, C4 (u16) 106 -> 129-139 us
template <int CB> constexpr uint32_t fold_code_bytes() { return kFoldChunksPerTile * 512u * CB; }
template <int CB> constexpr uint32_t fold_stage_bytes() { return fold_code_bytes<CB>() + kFoldChunksPerTile * 64u; }
// u8 full fold: results are staged in shared memory and written back by a storer warp
// with bulk (TMA) stores: codes, active words and the zeroed touch words of a tile.
template <int CB, bool WEIGH> constexpr bool fold_tma_out() { return !WEIGH; }
constexpr int kFoldOutStages = 2;
template <int CB, bool WEIGH> constexpr int fold_threads() {
  return 32 * (kFoldConsumerWarps + 1 + (fold_tma_out<CB, WEIGH>() ? 1 : 0));
}
template <int CB> constexpr uint32_t fold_out_stage_bytes() { return fold_code_bytes<CB>() + kFoldChunksPerTile * 64u; }
template <int CB, bool WEIGH = false> constexpr size_t fold_smem() {
  return (size_t)kFoldStages * fold_stage_bytes<CB>() +
         (fold_tma_out<CB, WEIGH>() ? (size_t)kFoldOutStages * fold_out_stage_bytes<CB>() + kFoldChunksPerTile * 64u : 0);
}

// WEIGH = true: read-only variant for window queries with k' < k on the closed pool
// (SURVEY §8(f) row 1): no touch fold, no preserveAT, no pool write-back.
// QL = log2(chunks per ATV) for g > 512 (g = 1024..4096, LPAL = 5): with 16 chunks per
// tile and chunks cc = warp, warp + 8, warp w always sees chunk w mod 2^QL of an ATV, so
// its per-lane constants stay fixed; the ATV weight is summed across the 2^QL warps
// with one packed shared-memory atomic (weight << 8 | arrival count).
template <int CB, int LPAL, bool WEIGH = false, int QL = 0>
// u8 fold: 2 CTAs per SM (84 registers) beat 3 (64 registers, operands rematerialised):
// C3 fold 63.2 -> 60.3 us (tools/gpu_fold1.sh)
#ifndef ASSE_FOLD_MINB1
#define ASSE_FOLD_MINB1 2
#endif
#ifndef ASSE_FOLD_MINB2
#define ASSE_FOLD_MINB2 2   // u16: 1 CTA per SM (133 registers) measured slower: C4 fold 117 vs 106 us
#endif
__global__ void __launch_bounds__(fold_threads<CB, WEIGH>(), CB == 1 ? ASSE_FOLD_MINB1 : ASSE_FOLD_MINB2) k_fold(FoldParams p) {
  using S = Swar<CB>;
  constexpr int NW = S::NW, EPW = S::EPW, EB = S::EB;
  constexpr uint32_t G = S::G;
  constexpr uint32_t EMASK = (EB == 8) ? 0xFFu : 0xFFFFu;
  constexpr uint32_t CODE_BYTES = fold_code_bytes<CB>();
  constexpr uint32_t STAGE_BYTES = fold_stage_bytes<CB>();
  constexpr uint32_t LPA = 1u << LPAL;
  constexpr uint32_t FIELD = 1u << (LPAL);        // bits per packed ATV weight: 8, 16, 32
  constexpr bool TOUT = fold_tma_out<CB, WEIGH>();
  constexpr uint32_t OUT_BYTES = fold_out_stage_bytes<CB>();
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kFoldStages], empty[kFoldStages];
  __shared__ __align__(8) uint64_t out_full[kFoldOutStages], out_empty[kFoldOutStages];
  uint8_t* const sout = smem + (size_t)kFoldStages * STAGE_BYTES;              // TOUT only
  uint8_t* const szero = sout + (size_t)kFoldOutStages * OUT_BYTES;            // TOUT only
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  // blocked tile range of this CTA (keeps each warp's (y, z) slab changes rare for AAT)
  const uint32_t n_tiles = (uint32_t)((p.n_chunks + kFoldChunksPerTile - 1) / kFoldChunksPerTile);
  const uint32_t per = (n_tiles + gridDim.x - 1) / gridDim.x;
  const uint32_t t0 = blockIdx.x * per;
  const uint32_t t1 = min(n_tiles, t0 + per);
  if (threadIdx.x == 0) {
    for (int st = 0; st < kFoldStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kFoldConsumerWarps);
    }
    if (TOUT)
      for (int st = 0; st < kFoldOutStages; ++st) {
        mbar_init(&out_full[st], kFoldConsumerWarps);
        mbar_init(&out_empty[st], 1);
      }
    mbar_fence_init();
  }
  if (TOUT) {
    for (uint32_t q = threadIdx.x; q < kFoldChunksPerTile * 16u; q += blockDim.x)
      reinterpret_cast<uint32_t*>(szero)[q] = 0u;
    fence_proxy_async_smem();
  }
  __syncthreads();
  if (t0 >= t1) return;
  if (TOUT && warp == kFoldConsumerWarps + 1) {     // storer warp: TMA bulk write-back
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (uint32_t i = 0; i < t1 - t0; ++i) {
        const uint32_t os = i % kFoldOutStages;
        mbar_wait(&out_full[os], (i / kFoldOutStages) & 1u);
        const uint32_t tile = t0 + i;
        const uint32_t nch = (uint32_t)umin64(kFoldChunksPerTile, p.n_chunks - (uint64_t)tile * kFoldChunksPerTile);
        const uint8_t* src = sout + (size_t)os * OUT_BYTES;
        bulk_s2g(reinterpret_cast<uint8_t*>(p.pool) + (size_t)tile * CODE_BYTES, src, nch * 512u * CB, pol);
        bulk_s2g(p.active + (size_t)tile * kFoldChunksPerTile * 16u, src + CODE_BYTES, nch * 64u, pol);
        bulk_s2g(p.touch_zero + (size_t)tile * kFoldChunksPerTile * 16u, szero, nch * 64u, pol);
        bulk_commit();
        bulk_wait_read0();                          // out stage may be rewritten
        mbar_arrive(&out_empty[os]);
      }
      bulk_wait0();                                 // writes complete before the kernel ends
    }
    return;
  }
  if (warp == kFoldConsumerWarps) {                 // producer warp: TMA bulk loads
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const uint64_t keep = policy_evict_last();
      for (uint32_t i = 0; i < t1 - t0; ++i) {
        const uint32_t st = i % kFoldStages;
        if (i >= kFoldStages) mbar_wait(&empty[st], ((i / kFoldStages) - 1) & 1u);
        const uint32_t tile = t0 + i;
        const uint32_t nch = (uint32_t)umin64(kFoldChunksPerTile, p.n_chunks - (uint64_t)tile * kFoldChunksPerTile);
        uint8_t* dst = smem + (size_t)st * STAGE_BYTES;
        mbar_expect_tx(&full[st], nch * (512u * CB + (WEIGH ? 0u : 64u)));
        bulk_g2s(dst, reinterpret_cast<const uint8_t*>(p.pool) + (size_t)tile * CODE_BYTES, nch * 512u * CB,
                 &full[st], pol);
        if (!WEIGH)
          bulk_g2s(dst + CODE_BYTES, p.touch_src + (size_t)tile * kFoldChunksPerTile * 16u, nch * 64u,
                   &full[st], keep);
      }
    }
    return;
  }
  const uint32_t lia = lane & (LPA - 1u);           // lane within its chunk of the ATV
  const uint32_t two_k = 2u * p.k;
  const uint32_t C0 = *p.C0;
  const uint32_t qoff = (QL > 0) ? 512u * (warp & ((1u << QL) - 1u)) : 0u;   // chunk offset in the ATV
  __shared__ uint32_t s_wacc[kFoldStages][kFoldChunksPerTile];
  if (QL > 0) {
    for (uint32_t q = threadIdx.x; q < kFoldStages * kFoldChunksPerTile; q += 32 * kFoldConsumerWarps)
      (&s_wacc[0][0])[q] = 0;
    asm volatile("bar.sync 1, %0;" :: "r"(32 * kFoldConsumerWarps));   // consumer warps only
  }

  // ---- per-lane, per-element constants (positions i = 16*lia + e), computed once
  uint32_t CLK[NW], LO1[NW], HI1[NW], LO2[NW], HI2[NW], LE1[NW], HE1[NW], LE2[NW], HE2[NW];
  uint32_t swept_mask = 0;  // bit q: word q holds ATs of a block swept for t+1
#pragma unroll
  for (int q = 0; q < NW; ++q) {
    CLK[q] = LO1[q] = HI1[q] = LO2[q] = HI2[q] = LE1[q] = HE1[q] = LE2[q] = HE2[q] = 0;
#pragma unroll
    for (int e = 0; e < EPW; ++e) {
      const uint32_t i = qoff + 16u * lia + (uint32_t)(q * EPW + e);
      uint32_t blk = (p.a > 0) ? min(i / p.a, two_k - 1u) : two_k - 1u;  // A7
      uint32_t clk = (C0 + blk) % two_k;
      uint32_t lo1, hi1 = clk, lo2, hi2;
      if (clk + 1u >= p.kp) { lo1 = clk + 1u - p.kp; lo2 = S::EMPTY_LO; hi2 = 0; }
      else { lo1 = 0; lo2 = clk + 1u + two_k - p.kp; hi2 = two_k - 1u; }
      // Alg. 2 for the new ACT of slice t+1
      uint32_t nclk = (clk + 1u == two_k) ? 0u : clk + 1u;
      uint32_t le1 = S::EMPTY_LO, he1 = 0, le2 = S::EMPTY_LO, he2 = 0;
      if (nclk == 0) { le1 = 0; he1 = p.k; }                                   // 0 <= at <= k
      else if (nclk == p.k) { le1 = p.k; he1 = two_k - 1u; le2 = 0; he2 = 0; } // k..2k-1 and 0
      if (le1 <= he1 || le2 <= he2) swept_mask |= 1u << q;
      const uint32_t sh = (uint32_t)e * EB;
      const uint32_t gbit = 1u << (EB - 1);
      CLK[q] |= clk << sh;
      LO1[q] |= lo1 << sh; HI1[q] |= (hi1 | gbit) << sh;
      LO2[q] |= lo2 << sh; HI2[q] |= (hi2 | gbit) << sh;
      if (CB == 1) {
        LE1[q] |= le1 << sh; HE1[q] |= (he1 | gbit) << sh;
        LE2[q] |= le2 << sh; HE2[q] |= (he2 | gbit) << sh;
      }
    }
  }
  swept_mask = __reduce_or_sync(0xFFFFFFFFu, swept_mask);   // warp-uniform per word
  uint32_t TWOK = 0;
#pragma unroll
  for (int e = 0; e < EPW; ++e) TWOK |= two_k << (e * EB);

  constexpr int LW = NW;                            // uint32 code words per lane
  const uint64_t pol = policy_evict_first();
  const uint32_t tshift = (lane & 1u) << 4;
  const uint32_t fshift = (lane >> LPAL) * FIELD;   // this lane's ATV field in the packed sum
  const uint32_t E = 1u << p.c;
  uint4* const gpool = reinterpret_cast<uint4*>(p.pool) + lane * (LW / 4);
  uint32_t* const gact = p.active + (lane >> 1);
  uint32_t* const gzero = p.touch_zero + (lane >> 1);
  unsigned long long aat_acc = 0;
  uint32_t aat_yz = 0xFFFFFFFFu;
  uint32_t nsup = 0;

  for (uint32_t i = 0; i < t1 - t0; ++i) {
    const uint32_t st = i % kFoldStages;
    mbar_wait(&full[st], (i / kFoldStages) & 1u);
    const uint32_t tile = t0 + i;
    const uint32_t nch = (uint32_t)umin64(kFoldChunksPerTile, p.n_chunks - (uint64_t)tile * kFoldChunksPerTile);
    const uint8_t* sbase = smem + (size_t)st * STAGE_BYTES;
    const uint4* scodes = reinterpret_cast<const uint4*>(sbase) + lane * (LW / 4);
    const uint32_t os = i % kFoldOutStages;
    uint4* ocodes = reinterpret_cast<uint4*>(sout + (size_t)os * OUT_BYTES) + lane * (LW / 4);
    uint32_t* oact = reinterpret_cast<uint32_t*>(sout + (size_t)os * OUT_BYTES + CODE_BYTES) + (lane >> 1);
    if (TOUT && i >= kFoldOutStages) mbar_wait(&out_empty[os], ((i / kFoldOutStages) - 1) & 1u);
    const uint32_t* stouch = reinterpret_cast<const uint32_t*>(sbase + CODE_BYTES) + (lane >> 1);
    for (uint32_t cc = warp; cc < nch; cc += kFoldConsumerWarps) {
      const uint32_t ch = tile * kFoldChunksPerTile + cc;
      uint32_t cur[LW];
#pragma unroll
      for (int v4 = 0; v4 < LW / 4; ++v4) {
        const uint4 t4 = scodes[cc * (32u * LW / 4) + v4];
        cur[4 * v4 + 0] = t4.x; cur[4 * v4 + 1] = t4.y; cur[4 * v4 + 2] = t4.z; cur[4 * v4 + 3] = t4.w;
      }
      const uint32_t field = WEIGH ? 0u : (stouch[cc * 16u] >> tshift) & 0xFFFFu;
      uint32_t v[LW];
      uint32_t accbits = 0;
      bool changed = false;
#pragma unroll
      for (int q = 0; q < NW; ++q) {
        // SetAT fold via PRMT: element e takes CLK's element when its touch bit is set
        uint32_t sel;
        if (CB == 1) {
          const uint32_t f = (q <= 2) ? (field << (2 - q)) : (field >> (q - 2));
          sel = 0x3210u | (f & 0x4444u);
        } else {
          sel = 0x3210u | (((field >> q) & 0x0101u) * 0x44u);
        }
        uint32_t x = WEIGH ? cur[q] : __byte_perm(cur[q], CLK[q], sel);
        // checkAT (Alg. 1): two intervals of the cyclic window
        const uint32_t vx = x | G;
        const uint32_t act = (in_range(vx, x, LO1[q], HI1[q]) | in_range(vx, x, LO2[q], HI2[q])) & G;
        accbits |= act >> ((CB == 1 ? 7 : 15) - q);
        // preserveAT for slice t+1 (Alg. 2), only in words holding swept blocks
        if (!WEIGH && (swept_mask & (1u << q))) {
          uint32_t er;
          if (CB == 1) {
            er = (in_range(vx, x, LE1[q], HE1[q]) | in_range(vx, x, LE2[q], HE2[q])) & G;
          } else {
            // u16: sweeps are rare (a = 0 sweeps whole ATVs every k slices), so the Alg. 2
            // intervals are derived here from the block ACT instead of held in registers:
            // new ACT 0 (clk = 2k-1) erases [0, k]; new ACT k (clk = k-1) erases [k, 2k-1] and 0
            const uint32_t ONE = 0x00010001u;
            const uint32_t d0 = CLK[q] ^ ((two_k - 1u) * ONE), dk = CLK[q] ^ ((p.k - 1u) * ONE);
            const uint32_t eq0 = ~((d0 | G) - ONE) & G, eqk = ~((dk | G) - ONE) & G;
            const uint32_t in0k = in_range(vx, x, 0u, (p.k * ONE) | G);
            const uint32_t inkk = in_range(vx, x, p.k * ONE, ((two_k - 1u) * ONE) | G) | in_range(vx, x, 0u, G);
            er = ((eq0 & in0k) | (eqk & inkk)) & G;
          }
          const uint32_t m = (er >> (EB - 1)) * EMASK;   // guard bit -> whole-element mask
          x = (x & ~m) | (TWOK & m);
        }
        changed |= (x != cur[q]);
        v[q] = x;
      }
      if (TOUT) {            // staged for the storer warp's bulk write-back
#pragma unroll
        for (int w4 = 0; w4 < LW / 4; ++w4)
          ocodes[cc * (32u * LW / 4) + w4] = make_uint4(v[4 * w4], v[4 * w4 + 1], v[4 * w4 + 2], v[4 * w4 + 3]);
      } else if (!WEIGH && changed) {   // write back only the lane slices that changed
#pragma unroll
        for (int w4 = 0; w4 < LW / 4; ++w4)
          st_pool(gpool + (size_t)ch * (32u * LW / 4) + w4,
                  make_uint4(v[4 * w4], v[4 * w4 + 1], v[4 * w4 + 2], v[4 * w4 + 3]), pol);
      }
      // active word = even-lane bits | odd-lane bits shifted into the free positions
      const uint32_t other = __shfl_xor_sync(0xFFFFFFFFu, accbits, 1);
      if ((lane & 1u) == 0) {
        const uint32_t aw = (CB == 1) ? (accbits | (other << 4)) : (accbits | (other << 8));
        if (TOUT) {
          oact[cc * 16u] = aw;
        } else {
          gact[(size_t)ch * 16u] = aw;
          if (!WEIGH) gzero[(size_t)ch * 16u] = 0u;
        }
      }
      // |ATV|^{k'} of every ATV in the chunk with one warp reduction: each ATV's
      // lanes add into their own FIELD-bit slot (max 16*LPA fits the slot)
      const uint32_t cnt = __popc(accbits);   // the guard bits of every word, gathered into 16 distinct bits
      const uint32_t packed = __reduce_add_sync(0xFFFFFFFFu, cnt << fshift);
      const uint32_t w = (FIELD == 32) ? packed : ((packed >> fshift) & ((1u << FIELD) - 1u));
      uint32_t tot;
      if (LPAL == 5) tot = packed;
      else if (LPAL == 4) tot = (packed & 0xFFFFu) + (packed >> 16);
      else tot = (packed & 0xFFu) + ((packed >> 8) & 0xFFu) + ((packed >> 16) & 0xFFu) + (packed >> 24);
      const uint32_t atv = (QL > 0) ? (ch >> QL) : (ch << (5 - LPAL)) + (lane >> LPAL);
      const uint32_t yz = atv >> p.c;
      bool is_super;
      if (QL > 0) {
        is_super = false;
        if (lane == 0) {
          const uint32_t add = (w << 8) | 1u;
          const uint32_t nv = atomicAdd(&s_wacc[st][cc >> QL], add) + add;
          if ((nv & 0xFFu) == (1u << QL)) {       // last of the ATV's chunks
            s_wacc[st][cc >> QL] = 0;             // stage slot reused after the empty barrier
            is_super = (nv >> 8) >= p.w_theta;
          }
        }
      } else {
        is_super = (lia == 0 && w >= p.w_theta);
      }
      if (is_super) {                              // super ATV
        const uint32_t xcol = atv & (E - 1u);
        const uint32_t slot = atomicAdd(p.sa_cnt + yz, 1u);
        p.sa_list[(size_t)yz * E + slot] = xcol;
        atomicOr(p.sa_bits + (atv >> 5), 1u << (xcol & 31u));
        nsup++;
      }
      // AAT: the whole chunk lies in one (y, z) slab (E*g >= 512)
      if (yz != aat_yz) {
        if (lane == 0 && aat_acc) atomicAdd(p.aat + aat_yz, aat_acc);
        aat_yz = yz;
        aat_acc = 0;
      }
      aat_acc += tot;
    }
    if (TOUT) fence_proxy_async_smem();             // staged writes -> async-proxy reads
    __syncwarp();
    if (lane == 0) {
      if (TOUT) mbar_arrive(&out_full[os]);
      mbar_arrive(&empty[st]);
    }
  }
  if (lane == 0 && aat_acc) atomicAdd(p.aat + aat_yz, aat_acc);
  nsup = __reduce_add_sync(0xFFFFFFFFu, nsup);
  if (lane == 0 && nsup) atomicAdd(p.n_super, nsup);
}

// ---------------------------------------------------------------- restore

struct RestoreParams {
  const uint32_t* sa_cnt;   // [r*F]
  const uint32_t* sa_list;  // [r*F][E]
  const uint32_t* sa_bits;  // [r*F][E/32]
  uint32_t* ws;             // join workspace: (F * parts) CTAs x 2 buffers x ws_cap
  uint64_t ws_cap;
  uint32_t parts;           // CTAs per frame: row 0's candidates are split among them
  uint32_t* cand;           // out: candidates as mangled values h = (LBS << u) | z
  uint32_t* n_cand;         // out: |CSIP|
  uint32_t* overflow;       // out: 1 if CSIP or a join level exceeded its capacity
  uint32_t max_cand;
  uint32_t r, u, c, W, F;
  uint32_t shift[kMaxR];    // (s*y) mod W
  uint32_t ov[kMaxR];       // bits of x_y already fixed by rows < y
  uint32_t nfree[kMaxR];    // c - popc(ov[y])
  uint32_t use_enum_max[kMaxR];  // enumerate the 2^nfree completions when 2^nfree <= this * |SA|
  uint8_t freepos[kMaxR][32];    // free bit positions of x_y
  // the free positions as two ascending runs: completion bits [0, n1) shift up by sh1
  // (= freepos[0]), bits [n1, nf) by sh2 (= freepos[n1] - n1)
  uint8_t dep_n1[kMaxR], dep_sh1[kMaxR], dep_sh2[kMaxR];
  // Alg. 5 / Eq. 5 for every restored candidate (fused)
  const uint32_t* active;        // active bits, wpa words per ATV
  const unsigned long long* aat; // AAT[y][z]
  void* reports;                 // asse_report per CSIP slot
  uint32_t* keys;                // ip per slot (device-wide sort)
  uint32_t* vals;                // slot index (device-wide sort)
  uint64_t A_inv;
  uint32_t mangle_p;             // 1: f^{-1} by mod-p cycle walking
  uint32_t g, wpa;
  uint32_t z_base;               // global index of local frame 0 (option S: rank * F_local)
  uint32_t sys_fence;            // option S: publish the reports to peers (system-scope fence)
  double theta, cells;           // cells = g * 2^c
};

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
struct ReportDev { uint32_t ip, nat; double estimate; uint32_t flags, pad; };

__device__ __forceinline__ uint32_t place_row(uint32_t x, uint32_t sh, uint32_t W) {
  // LBS bits (sh + j) mod W <- x[j] (P:324 wrap-around)
  uint64_t P = (uint64_t)x << sh;
  uint32_t wmask = (W >= 32) ? 0xFFFFFFFFu : ((1u << W) - 1u);
  return (uint32_t)((P | (P >> W)) & wmask);
}

// Alg. 4 per frame z (parts CTAs, each taking every parts-th row-0 candidate): CSIP_z = {LBS : x_y(LBS) in SA(y, z) for all y}.
// The r-fold product of P:364 is evaluated as a join: rows are added one at a time,
// and a partial LBS only survives when every duplicate position agrees,
// which yields exactly the tuples that pass Alg. 4's check (A16). Row y either scans
// SA(y,z) comparing the already-fixed bits, or enumerates the 2^nfree completions of
// x_y and tests SA membership — whichever is fewer probes.
constexpr uint32_t kPartSmem = 2048;   // partial LBS kept in shared memory per level buffer

#ifdef ASSE_RESTORE_PROF
__device__ unsigned long long g_restore_prof[4096][8];   // tools only: per-CTA globaltimer marks
#define RPROF(k) do { if (threadIdx.x == 0 && blockIdx.x < 4096) { unsigned long long t_; \
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); g_restore_prof[blockIdx.x][k] = t_; } } while (0)
#else
#define RPROF(k) ((void)0)
#endif
// Latency (per-CTA globaltimer marks, tools/restore_timeline.py, C3): prologue 1.8 us, rows
// 0-2 ~1.3 us each, the last row with Alg. 5 5.1 us, when each row took three CTA barriers,
// a dependent constant-bank load per free bit of the enumeration and row 0's list load
// after the prologue, and the last row waited for its global slot before loading the NAT
// words. Now: one barrier per row (three rotating counters), the free bits deposited as at
// most two contiguous runs (host-derived; a loop otherwise), row 0's first 32 options of the
// part prefetched in the prologue, the NAT loads issued while the slot atomic is in flight.
__global__ void __launch_bounds__(512, 2) k_restore(RestoreParams p) {   // 2 CTAs per SM: one wave of F x parts
  extern __shared__ uint32_t s_bits[];  // r * E/32 words of SA(y, z) membership
  __shared__ uint32_t s_part[2][kPartSmem];
  __shared__ uint32_t s_nsa[kMaxR];
  __shared__ uint32_t s_cnt[3];         // output count of row y: s_cnt[y % 3]
  __shared__ uint32_t s_pre[32];        // row 0 (list scan): options part + j * parts, j < 32
  __shared__ double s_up;
  const uint32_t z = blockIdx.x / p.parts;
  const uint32_t part = blockIdx.x % p.parts;
  const uint32_t E = 1u << p.c;
  const uint32_t ew = (E + 31u) >> 5;
  const uint32_t cmask = (p.c >= 32) ? 0xFFFFFFFFu : ((1u << p.c) - 1u);
  // partial buffers: slots < kPartSmem in shared memory, the rest in the global workspace
  uint32_t* gbuf[2] = {p.ws + (size_t)blockIdx.x * 2 * p.ws_cap,
                       p.ws + (size_t)blockIdx.x * 2 * p.ws_cap + p.ws_cap};
  RPROF(0);
  pdl_wait();                                         // k_fold's SA lists, bits, AAT, active bits
  RPROF(1);
#ifdef ASSE_RESTORE_EMPTY
  pdl_trigger();                                      // tools only: the restore's share of the step
  return;
#endif
  // prologue, one round trip: |SA(y, z)|, row 0's prefetched options, UP, the SA bits
  if (threadIdx.x < p.r) s_nsa[threadIdx.x] = __ldcg(p.sa_cnt + threadIdx.x * p.F + z);
  if (threadIdx.x >= 32 && threadIdx.x < 64) {
    const uint32_t j = threadIdx.x - 32, o = part + j * p.parts;
    s_pre[j] = (o < E) ? __ldcg(p.sa_list + (size_t)z * E + o) : 0u;
  }
  if (threadIdx.x == 64) {
    // UP_{k'}^{z} = prod_y AAT[y][z] / (g 2^c) (Eq. 4), same product order as the oracle
    double up = 0.0;
    for (uint32_t y = 0; y < p.r; ++y) {
      const double P = (double)__ldcg(p.aat + y * p.F + z) / p.cells;
      up = (y == 0) ? P : up * P;
    }
    s_up = up;
  }
  if (threadIdx.x == 96) {
    s_cnt[0] = 0; s_cnt[1] = 0; s_cnt[2] = 0;
    s_part[0][0] = 0;                                 // the empty partial LBS
  }
  for (uint32_t q = threadIdx.x; q < p.r * ew; q += blockDim.x) {
    const uint32_t y = q / ew, w = q % ew;
    s_bits[q] = __ldcg(p.sa_bits + ((size_t)y * p.F + z) * ew + w);
  }
  __syncthreads();
  RPROF(2);
#ifdef ASSE_RESTORE_PROLOGUE_ONLY
  pdl_trigger();                                      // tools only: launch + prologue share
  return;
#endif
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t n_in = 1;
  for (uint32_t y = 0; y < p.r; ++y) {
    const uint32_t nsa = s_nsa[y];
    if (n_in == 0 || nsa == 0) break;                 // uniform across the CTA
    uint32_t* const cnt = &s_cnt[y % 3];              // zero (set two rows ago)
    if (threadIdx.x == 0) s_cnt[(y + 1) % 3] = 0;     // next row's; last read as n_in before row y-1
    const bool last = (y + 1 == p.r);
    const uint32_t nf = p.nfree[y];
    const bool use_enum = ((1ull << nf) <= (uint64_t)p.use_enum_max[y] * nsa);
    const uint64_t n_opt = use_enum ? (1ull << nf) : (uint64_t)nsa;
    // row 0 (single empty partial): this CTA takes options part, part + parts, ...
    const uint64_t per = (y == 0) ? (n_opt > part ? (n_opt - part + p.parts - 1) / p.parts : 0) : n_opt;
    const uint64_t total = (uint64_t)n_in * per;
    const uint32_t ib = y & 1u, ob = (y + 1) & 1u;
    const uint32_t* sal = p.sa_list + ((size_t)y * p.F + z) * E;
    const uint32_t* bits = s_bits + y * ew;
    const uint32_t sh = p.shift[y], ovy = p.ov[y];
    const uint32_t dn1 = p.dep_n1[y], ds1 = p.dep_sh1[y], ds2 = p.dep_sh2[y];
    const uint64_t rounded = (total + 31u) & ~31ull;
    for (uint64_t idx = threadIdx.x; idx < rounded; idx += blockDim.x) {
      bool ok = false;
      uint32_t nl = 0;
      if (idx < total) {
        // (partial, option) of this probe: 32-bit division whenever the level fits 32 bits
        uint32_t pi, jj;
        if (total <= 0xFFFFFFFFull) { pi = (uint32_t)idx / (uint32_t)per; jj = (uint32_t)idx - pi * (uint32_t)per; }
        else { pi = (uint32_t)(idx / per); jj = (uint32_t)(idx % per); }
        const uint32_t L = (pi < kPartSmem) ? s_part[ib][pi] : gbuf[ib][pi - kPartSmem];
        const uint32_t sub = (y == 0) ? part + jj * p.parts : jj;
        const uint64_t D = (uint64_t)L | ((uint64_t)L << p.W);
        const uint32_t xk = (uint32_t)(D >> sh) & cmask;
        uint32_t x;
        if (use_enum) {
          // the completion sub's bits go to the free positions of x_y (ascending), which form
          // at most two runs: the window is a cyclic interval and the fixed LBS bits a growing
          // one (host-checked; tests/test_host_logic.py over every admissible geometry)
          const uint32_t m1 = (1u << dn1) - 1u;     // dn1 <= nf <= c < 32
          x = (xk & ovy) | ((sub & m1) << ds1) | ((sub & ~m1) << ds2);
          ok = (bits[x >> 5] >> (x & 31u)) & 1u;
        } else {
          x = (y == 0 && jj < 32) ? s_pre[jj] : __ldcg(sal + sub);
          ok = ((x ^ xk) & ovy) == 0;
        }
        nl = L | place_row(x, sh, p.W);
      }
      // warp-aggregated append
      const uint32_t m = __ballot_sync(0xFFFFFFFFu, ok);
      if (!m) continue;
      const uint32_t rank = __popc(m & lt);
      const uint32_t leader = __ffs(m) - 1;
      if (!last) {
        uint32_t base = 0;
        if (lane == leader) base = atomicAdd(cnt, __popc(m));
        base = __shfl_sync(0xFFFFFFFFu, base, leader);
        if (!ok) continue;
        const uint32_t slot = base + rank;
        if (slot < kPartSmem) s_part[ob][slot] = nl;
        else if (slot < kPartSmem + p.ws_cap) gbuf[ob][slot - kPartSmem] = nl;
        else *p.overflow = 1u;
        continue;
      }
      // a restored candidate: the warp's slots are reserved first, the NAT words load while
      // the atomic is in flight (the slot is only needed for the stores)
      uint32_t base = 0;
      if (lane == leader) base = atomicAdd(p.n_cand, __popc(m));
      uint32_t h = 0, nat = 0, flags = 0, ip = 0;
      double est = 0.0;
      if (ok) {
        // f(ip) = (LBS << u) | z, ip = A^{-1} f
        h = (p.u ? (nl << p.u) : nl) | (p.z_base + z);
        // Alg. 5 NAT: ATs active in all r ATVs of the candidate, 4 x 16 B of
        // every row per batch, all loads issued before the AND (g = 512: one batch)
        const uint64_t DL = (uint64_t)nl | ((uint64_t)nl << p.W);
        const uint4* rows[kMaxR];
#pragma unroll
        for (int yy = 0; yy < kMaxR; ++yy) {
          const uint32_t xx = (yy < (int)p.r) ? (uint32_t)(DL >> p.shift[yy]) & cmask : 0u;
          rows[yy] = reinterpret_cast<const uint4*>(p.active + ((((size_t)yy * p.F + z) << p.c) | xx) * p.wpa);
        }
        const uint32_t nw4 = p.wpa / 4;
        for (uint32_t w0 = 0; w0 < nw4; w0 += 4) {
          uint4 a[4][kMaxR];
#pragma unroll
          for (int yy = 0; yy < kMaxR; ++yy)
#pragma unroll
            for (int k = 0; k < 4; ++k)
              a[k][yy] = (yy < (int)p.r && w0 + k < nw4) ? __ldcg(rows[yy] + w0 + k)
                                                        : make_uint4(~0u, ~0u, ~0u, ~0u);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            uint4 acc = a[k][0];
#pragma unroll
            for (int yy = 1; yy < kMaxR; ++yy) {
              acc.x &= a[k][yy].x; acc.y &= a[k][yy].y; acc.z &= a[k][yy].z; acc.w &= a[k][yy].w;
            }
            if (w0 + k < nw4) nat += __popc(acc.x) + __popc(acc.y) + __popc(acc.z) + __popc(acc.w);
          }
        }
        // Eq. 5 (A19) in double; NAT == g -> +inf (A20)
        if (nat == p.g) est = __longlong_as_double(0x7FF0000000000000LL);
        else est = -(double)p.g * log((double)(p.g - nat) / ((double)p.g * (1.0 - s_up)));
        flags = (nat == p.g ? 1u : 0u) | (est >= p.theta ? 2u : 0u);
        ip = p.mangle_p ? walk_mod_p(p.A_inv, h) : (uint32_t)p.A_inv * h;   // f^{-1}
      }
      base = __shfl_sync(0xFFFFFFFFu, base, leader);
      if (!ok) continue;
      const uint32_t slot = base + rank;
      if (slot >= p.max_cand) { *p.overflow = 1u; continue; }
#ifdef ASSE_RESTORE_NO_NAT
      continue;                                       // tools only: the join without the report stores
#endif
      p.cand[slot] = h;
      ReportDev* R = reinterpret_cast<ReportDev*>(p.reports) + slot;
      R->ip = ip; R->nat = nat; R->estimate = est; R->flags = flags; R->pad = 0;
      p.keys[slot] = ip;
      p.vals[slot] = slot;
    }
    __syncthreads();
    RPROF(3 + (y < 3 ? y : 3));
    n_in = (uint32_t)min((uint64_t)*cnt, (uint64_t)kPartSmem + p.ws_cap);   // (last row: unused)
  }
  RPROF(7);
  if (p.sys_fence) __threadfence_system();
  pdl_trigger();
}

// Sort of CSIP by ip (A24) and the est >= theta subset (A21), |CSIP| read on the device:
//  * |CSIP| <= 2048: rank sort, one warp per element — CSIP ips are distinct (tuple <->
//    LBS bijection, A16), so an element's position is the number of smaller ips and its
//    position among the ABOVE_THETA reports counts the smaller flagged ips;
//  * larger: counters[5] = 1 and the bucket sort below runs (k_bs_*; in the end_slice graph
//    once a slice needed it, else from the host).
// counters: [0] n_cand, [4] n_above, [5] big.
constexpr int kSortThreads = 512;
constexpr uint32_t kRankCap = 2048;
constexpr int kSortBlocks = kRankCap / (kSortThreads / 32);   // 128: one warp per element

__global__ void __launch_bounds__(kSortThreads) k_sort(const ReportDev* __restrict__ rep, uint32_t* counters,
                                                       const uint32_t* n_ptr, uint32_t max_cand,
                                                       ReportDev* __restrict__ sorted,
                                                       ReportDev* __restrict__ above,
                                                       uint32_t* clock, uint32_t two_k) {
  struct Smem { uint32_t key[kRankCap]; uint32_t above[kRankCap / 32]; };
  __shared__ __align__(16) Smem sm;
  pdl_wait();                                          // k_restore's reports and |CSIP|
  // a9: the next slice's ACT base, advanced on the device (k_fold and k_restore of this
  // slice are complete), so no host-to-device copy precedes the next end_slice
  if (clock && blockIdx.x == 0 && threadIdx.x == 0) *clock = (*clock + 1u == two_k) ? 0u : *clock + 1u;
  const uint32_t n = min(*n_ptr, max_cand);
#ifdef ASSE_SORT_EMPTY
  return;                                              // tools only: the sort's share of the step
#endif
  if (n == 0) return;
  if (n > kRankCap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) counters[5] = 1u;
    return;
  }
  // rank sort
  const uint32_t first = blockIdx.x * (kSortThreads / 32);
  if (first >= n) return;                              // CTA without elements
  for (uint32_t j = threadIdx.x; j < kRankCap / 32; j += kSortThreads) sm.above[j] = 0;
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < n; j += kSortThreads) {
    const ReportDev r = rep[j];
    sm.key[j] = r.ip;
    if (r.flags & 2u) atomicOr(&sm.above[j >> 5], 1u << (j & 31u));
  }
  __syncthreads();
  const uint32_t q = first + (threadIdx.x >> 5);
  if (q >= n) return;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t k = sm.key[q];
  uint32_t r_all = 0, r_above = 0;
  for (uint32_t j = lane; j < n; j += 32) {
    const uint32_t less = sm.key[j] < k ? 1u : 0u;
    r_all += less;
    r_above += less & (sm.above[j >> 5] >> (j & 31u));
  }
  r_all = __reduce_add_sync(0xFFFFFFFFu, r_all);
  r_above = __reduce_add_sync(0xFFFFFFFFu, r_above);
  if (lane == 0) {
    const ReportDev r = rep[q];
    sorted[r_all] = r;
    if (r.flags & 2u) {
      above[r_above] = r;
      atomicAdd(counters + 4, 1u);
    }
  }
}

// Bucket sort of CSIP by ip (A24) for |CSIP| > kRankCap, with the est >= theta subset in the
// same order (A21). CSIP ips are distinct (A16), so placing every ip in the bucket of its top
// bits and ranking it among its bucket (number of smaller ips) is an exact sort; the ranks
// inside a bucket need no stability. B = 2^bits buckets (host-chosen, ~32 ips per bucket for
// uniformly spread ips; any distribution is still sorted exactly, a crowded bucket only
// costs time). |CSIP| is read on the device: every kernel does nothing when n <= kRankCap
// (k_sort's rank sort handled it).
struct BucketSortParams {
  const ReportDev* rep;   // reports in slot order
  const uint32_t* keys;   // ip per slot
  const uint32_t* vals;   // report slot per slot
  const uint32_t* n_ptr;
  uint32_t max_cand, B, shift;   // shift = 32 - log2(B)
  uint32_t* cnt;          // [B] ips per bucket (zeroed before k_bs_count)
  uint32_t* off;          // [B] first position of each bucket
  uint32_t* cur;          // [B] scatter cursors
  uint32_t* acnt;         // [B] flagged reports per bucket
  uint32_t* aoff;         // [B] first above-theta position of each bucket
  uint32_t* tk;           // [max_cand] keys in bucket order
  uint32_t* tv;           // [max_cand] slots in bucket order
  uint32_t* arank;        // [max_cand] per sorted position: rank among the flagged, or ~0
  uint32_t* pbkt;         // [max_cand] per sorted position: its bucket
  ReportDev* sorted;
  ReportDev* above;
  uint32_t* counters;
};

__device__ __forceinline__ uint32_t bs_n(const BucketSortParams& p) { return min(*p.n_ptr, p.max_cand); }

__global__ void __launch_bounds__(256) k_bs_count(BucketSortParams p) {
  const uint32_t n = bs_n(p);
  if (n <= kRankCap) return;
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x)
    atomicAdd(p.cnt + (p.keys[q] >> p.shift), 1u);
}

// exclusive scan of in[0..B) into out (and out2 if given) by one CTA of 1024 threads
__device__ __forceinline__ uint32_t bs_block_scan(const uint32_t* in, uint32_t* out, uint32_t* out2, uint32_t B) {
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t carry;
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < B; base += blockDim.x) {
    const uint32_t q = base + threadIdx.x;
    const uint32_t v = q < B ? in[q] : 0u;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= (uint32_t)o) incl += t;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      const uint32_t w = (lane < blockDim.x / 32) ? wsum[lane] : 0u;
      uint32_t wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, wi, o);
        if (lane >= (uint32_t)o) wi += t;
      }
      wsum[lane] = wi - w;                              // exclusive prefix of the warp sums
    }
    __syncthreads();
    const uint32_t ex = carry + wsum[wid] + incl - v;
    if (q < B) {
      out[q] = ex;
      if (out2) out2[q] = ex;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = ex + v;
    __syncthreads();
  }
  return carry;
}

__global__ void __launch_bounds__(1024) k_bs_scan(BucketSortParams p) {
  if (bs_n(p) <= kRankCap) return;
  bs_block_scan(p.cnt, p.off, p.cur, p.B);
}

__global__ void __launch_bounds__(256) k_bs_scatter(BucketSortParams p) {
  const uint32_t n = bs_n(p);
  if (n <= kRankCap) return;
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const uint32_t k = p.keys[q];
    const uint32_t pos = atomicAdd(p.cur + (k >> p.shift), 1u);
    p.tk[pos] = k;
    p.tv[pos] = p.vals[q];
  }
}

// one warp per bucket: rank every ip among its bucket (all ips and the flagged ones)
constexpr uint32_t kBsWarps = 8, kBsCap = 512;   // keys staged per warp in shared memory
constexpr uint32_t kBsMaxLgB = 16, kBsMaxB = 1u << kBsMaxLgB;   // buckets at most
constexpr int kBsKernels = 6;
__global__ void __launch_bounds__(32 * kBsWarps) k_bs_bucket(BucketSortParams p) {
  __shared__ uint32_t skey[kBsWarps][kBsCap];
  __shared__ uint32_t sflag[kBsWarps][kBsCap / 32];
  const uint32_t n = bs_n(p);
  if (n <= kRankCap) return;
  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  const uint32_t b = blockIdx.x * kBsWarps + w;
  if (b >= p.B) return;
  const uint32_t s = p.cnt[b], o = p.off[b];
  const bool staged = s <= kBsCap;
  uint32_t nflag = 0;
  if (staged) {
    for (uint32_t j = lane; j < kBsCap / 32; j += 32) sflag[w][j] = 0;
    __syncwarp();
    for (uint32_t j = lane; j < s; j += 32) {
      skey[w][j] = p.tk[o + j];
      if (p.rep[p.tv[o + j]].flags & 2u) atomicOr(&sflag[w][j >> 5], 1u << (j & 31u));
    }
    __syncwarp();
  }
  for (uint32_t j0 = 0; j0 < s; j0 += 32) {
    const uint32_t j = j0 + lane;
    uint32_t kj = 0, r = 0, ra = 0;
    bool fj = false;
    if (j < s) {
      kj = staged ? skey[w][j] : p.tk[o + j];
      const ReportDev rj = p.rep[p.tv[o + j]];
      fj = (rj.flags & 2u) != 0;
      for (uint32_t i = 0; i < s; ++i) {
        const uint32_t ki = staged ? skey[w][i] : p.tk[o + i];
        const uint32_t less = ki < kj ? 1u : 0u;
        r += less;
        const uint32_t fi = staged ? (sflag[w][i >> 5] >> (i & 31u)) & 1u
                                   : ((p.rep[p.tv[o + i]].flags >> 1) & 1u);
        ra += less & fi;
      }
      const uint32_t pos = o + r;
      p.sorted[pos] = rj;
      p.arank[pos] = fj ? ra : 0xFFFFFFFFu;
      p.pbkt[pos] = b;
    }
    nflag += __popc(__ballot_sync(0xFFFFFFFFu, fj));
  }
  if (lane == 0) p.acnt[b] = nflag;
}

__global__ void __launch_bounds__(1024) k_bs_scan2(BucketSortParams p) {
  if (bs_n(p) <= kRankCap) return;
  const uint32_t tot = bs_block_scan(p.acnt, p.aoff, nullptr, p.B);
  if (threadIdx.x == 0) {
    p.counters[4] = tot;
    p.counters[5] = 0u;                                 // handled on the device
  }
}

__global__ void __launch_bounds__(256) k_bs_above(BucketSortParams p) {
  const uint32_t n = bs_n(p);
  if (n <= kRankCap) return;
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const uint32_t ar = p.arank[q];
    if (ar != 0xFFFFFFFFu) p.above[p.aoff[p.pbkt[q]] + ar] = p.sorted[q];
  }
}

// --------------------------------------------------------------- export

__global__ void k_export_u8(const uint8_t* __restrict__ in, uint16_t* __restrict__ out, uint64_t n) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n;
       q += (uint64_t)gridDim.x * blockDim.x)
    out[q] = in[q];
}

__global__ void k_fill_u8(uint8_t* p, uint8_t v, uint64_t n) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n;
       q += (uint64_t)gridDim.x * blockDim.x)
    p[q] = v;
}
__global__ void k_fill_u16(uint16_t* p, uint16_t v, uint64_t n) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n;
       q += (uint64_t)gridDim.x * blockDim.x)
    p[q] = v;
}

// ------------------------------------------------------------ multi-GPU

struct MergeParams {
  const uint4* touch[kMaxWorld];   // every rank's touch bitmap (peer-mapped)
  uint4* merged[kMaxWorld];        // every rank's merged bitmap (peer-mapped)
  uint32_t world;
  uint64_t lo, hi;                 // this rank's shard of uint4 words
};

// a5 (A26): OR of every rank's touch words in this rank's shard, stored to every
// rank's merged bitmap — reduce-scatter and all-gather in one pass over NVLink.
__global__ void __launch_bounds__(256) k_merge_or(MergeParams p) {
  for (uint64_t q = p.lo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < p.hi;
       q += (uint64_t)gridDim.x * blockDim.x) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (uint32_t w = 0; w < p.world; ++w) {
      uint4 v = __ldcv(p.touch[w] + q);
      acc.x |= v.x; acc.y |= v.y; acc.z |= v.z; acc.w |= v.w;
    }
    for (uint32_t w = 0; w < p.world; ++w) __stcg(p.merged[w] + q, acc);
  }
  // make this thread's peer stores visible system-wide before the kernel completes;
  // the following k_barrier release/acquire then orders them before every rank's fold
  __threadfence_system();
}

// a5, option S: rank d ORs every rank's touch words of its own frames into its local
// merged bitmap (a reduce-scatter over NVLink; frames of a row are contiguous).
struct MergeShardParams {
  const uint4* touch[kMaxWorld];   // every rank's (whole-geometry) touch bitmap
  uint4* merged;                   // this rank's merged bitmap (own frames only)
  uint32_t world;
  uint64_t row_local, row_global;  // uint4 words per row: own frames / all frames
  uint64_t frame_off;              // uint4 offset of the first own frame inside a row
  uint64_t n;                      // uint4 words of the local merged bitmap
};
__global__ void __launch_bounds__(256) k_merge_shard(MergeShardParams p) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < p.n;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t y = q / p.row_local, rest = q % p.row_local;
    const uint64_t gq = y * p.row_global + p.frame_off + rest;
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (uint32_t w = 0; w < p.world; ++w) {
      const uint4 v = __ldcv(p.touch[w] + gq);
      acc.x |= v.x; acc.y |= v.y; acc.z |= v.z; acc.w |= v.w;
    }
    p.merged[q] = acc;
  }
}

// Option S: gather every rank's published reports (count at byte 0, reports at byte
// 64 of its exchange buffer) into this rank's report array, with keys/values for the
// device-wide sort; counters[6] = total, counters[1] = overflow.
struct GatherParams {
  const uint8_t* xchg[kMaxWorld];
  uint32_t world, max_cand;
  ReportDev* rep;
  uint32_t* keys;
  uint32_t* vals;
  uint32_t* counters;
};
__global__ void __launch_bounds__(256) k_gather_peers(GatherParams p) {
  __shared__ uint32_t s_off[kMaxWorld + 1];
  if (threadIdx.x == 0) {
    uint32_t acc = 0;
    for (uint32_t w = 0; w < p.world; ++w) {
      s_off[w] = acc;
      acc += __ldcv(reinterpret_cast<const uint32_t*>(p.xchg[w]));
    }
    s_off[p.world] = acc;
    if (blockIdx.x == 0) {
      p.counters[6] = acc;
      if (acc > p.max_cand) p.counters[1] = 1u;
    }
  }
  __syncthreads();
  const uint32_t total = min(s_off[p.world], p.max_cand);
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < total; q += gridDim.x * blockDim.x) {
    uint32_t w = 0;
    while (q >= s_off[w + 1]) ++w;
    const ReportDev* src = reinterpret_cast<const ReportDev*>(p.xchg[w] + 64) + (q - s_off[w]);
    ReportDev r;
    r.ip = __ldcv(&src->ip); r.nat = __ldcv(&src->nat);
    r.estimate = __ldcv(&src->estimate); r.flags = __ldcv(&src->flags); r.pad = 0;
    p.rep[q] = r;
    p.keys[q] = r.ip;
    p.vals[q] = q;
  }
}

struct BarrierParams {
  uint32_t* pads[kMaxWorld];  // every rank's signal pad (peer-mapped)
  uint32_t world, rank, epoch;
};

// Cross-rank barrier over signal pads: publish `epoch` into slot [rank] of every peer's
// pad (release, system scope), then wait until every slot of our pad reached `epoch`
// (acquire). Called by one whole block of >= world threads.
constexpr uint64_t kBarrierTimeoutNs = 30ull * 1000000000ull;   // 30 s
__device__ __forceinline__ void barrier_ranks(uint32_t* const* pads, uint32_t world, uint32_t rank,
                                              uint32_t epoch) {
  const uint32_t w = threadIdx.x;
  __syncthreads();
  if (w < world) {
    uint32_t* dst = pads[w] + rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(dst), "r"(epoch) : "memory");
  }
  if (w < world) {
    const uint32_t* src = pads[rank] + w;
    uint32_t v;
    uint64_t t0 = 0;
    uint32_t spins = 0;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(src) : "memory");
      // watchdog: a rank that never arrives (a crashed peer, a protocol fault) ends the
      // kernel with an error after kBarrierTimeoutNs instead of hanging the GPU
      if ((++spins & 1023u) == 0) {
        uint64_t now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (t0 == 0) t0 = now;
        else if (now - t0 > kBarrierTimeoutNs) __trap();
      }
    } while ((int32_t)(v - epoch) < 0);
  }
  __syncthreads();
}

// Stream-ordered cross-GPU barrier (sync_mode 0). One process per GPU only: never launch
// several ranks' barriers on one GPU (nothing guarantees they run at the same time).
__global__ void k_barrier(BarrierParams p) { barrier_ranks(p.pads, p.world, p.rank, p.epoch); }

// asse_selftest_barrier: the ranks are the blocks of ONE cooperative launch (co-resident).
// Per epoch e every rank writes data[rank] = e, crosses the barrier, checks that it sees
// data[w] == e for every w (the release/acquire chain), and crosses a second barrier before
// the next epoch overwrites the data (reads ordered before the peers' next writes).
struct BarrierTestParams {
  BarrierParams bp;
  uint32_t* data;                  // [world] x 32 words
  unsigned long long* errors;
  uint32_t epochs;
};
__global__ void k_barrier_selftest(BarrierTestParams p) {
  const uint32_t rank = blockIdx.x, w = threadIdx.x;
  for (uint32_t e = 1; e <= p.epochs; ++e) {
    if (w == 0) p.data[rank * 32] = e;
    barrier_ranks(p.bp.pads, p.bp.world, rank, 2 * e - 1);
    if (w < p.bp.world) {
      const uint32_t v = *reinterpret_cast<volatile uint32_t*>(p.data + w * 32);
      if (v != e) atomicAdd(p.errors, 1ull);
    }
    barrier_ranks(p.bp.pads, p.bp.world, rank, 2 * e);
  }
}

}  // namespace asse
