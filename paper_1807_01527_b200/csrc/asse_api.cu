// asse_api.cu — C-ABI of libasse (include/asse.h): context, slice state machine,
// device memory, launches. Host code here only marshals arguments and sequences
// kernels; every step of the hot path runs in asse_kernels.cuh.
//
// P:n = PAPER.md line n; A<n> = reading n of DESIGN.md §2.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "asse.h"
#include "asse_kernels.cuh"
#include "asse_scan_bin.cuh"
#include "asse_scan_own.cuh"

using namespace asse;

namespace {

// NVTX ranges around every public entry point that enqueues device work (tracing: nsys /
// ncu --nvtx show the library's phases on the timeline; no-ops without a tool attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

struct Ctx {
  asse_config cfg{};
  // geometry
  uint32_t F = 0, E = 0, W = 0, two_k = 0, kp = 0, a = 0, b = 0, cb = 1, wpa = 0;
  uint32_t w_theta = 0, lpa_log2 = 0, q_log2 = 0;
  uint32_t shift[kMaxR] = {0};
  uint64_t n_atv = 0, n_at = 0;       // this context's ATVs / ATs (its frames in option S)
  uint64_t n_atv_full = 0;            // whole geometry (touch bitmap)
  uint32_t Fl = 0, z_base = 0;        // local frames and global index of local frame 0
  bool shard = false;                 // option S (frame-sharded)
  // keys (A14)
  uint64_t A = 0, A_inv = 0;
  uint64_t K_bh = 0;
  // clock (A3)
  uint32_t C0 = 0;
  uint64_t t = 0;
  // device
  int device = 0, sms = 148;
  int scan_grid = 0, fold_grid = 0;   // resident CTAs (SMs x occupancy)
  // binned scan (asse_scan_bin.cuh): one owner CTA per SM, shared-memory bitmap slices
  int scan_variant = 0;               // 0 auto, 1 k_scan (direct RED), 2 k_scan_bin
  bool bin_ok = false;                // geometry fits the SMs' shared memory
  uint32_t bin_G = 0, bin_wpo = 0, bin_rr = 1, bin_tile = 0;   // rows via RED (measured best: 1), tile bytes
  uint32_t bin_inv = 0;
  size_t bin_smem = 0;
  uint32_t* bin_queue = nullptr;      // [NB][G][QCAP]
  uint32_t* bin_sync = nullptr;       // [2 NB]
  // packet-owned scan (asse_scan_own.cuh): owner = (frame, word group of the AT position)
  bool own_ok = false;
  uint32_t own_O = 0, own_lg_ngrp = 0, own_lg_wg = 0, own_tile = 0;
  size_t own_smem = 0;
  uint2* own_queue = nullptr;         // [NB][O][QG][QCAP]
  uint32_t* own_sync = nullptr;      // two sets of the packet-owned scan's counters (launch parity)
  uint32_t own_parity = 0;
  cudaStream_t stream = nullptr, copy_stream = nullptr;
  cudaStream_t d2h_stream = nullptr;  // result copies of end_slice (off the context stream)
  cudaEvent_t ev_done = nullptr;      // end of a slice's kernels on the context stream
  bool collect_pending = false;       // ev_collect recorded: the next end_slice waits on it
  void* pool = nullptr;
  uint32_t* touch_own = nullptr;
  uint32_t* touch = nullptr;        // where k_scan records (own or peer-mapped)
  uint32_t* merged = nullptr;       // world > 1: merged bitmap of this rank
  uint32_t* active = nullptr;
  unsigned long long* aat = nullptr;
  uint32_t* sa_cnt = nullptr;
  uint32_t* sa_list = nullptr;
  uint32_t* sa_bits = nullptr;
  uint32_t* counters = nullptr;     // [0] n_cand [1] overflow [2] n_above [3] n_super [4] n_sel [5] big
  void* scratch = nullptr;          // aat | sa_cnt | counters | sa_bits, zeroed per slice
  size_t scratch_bytes = 0;
  RestoreParams rp0{};              // geometry part of the restore parameters
  uint32_t* d_clock = nullptr;      // device copy of C0, refreshed from h_clock per slice
  uint32_t* h_clock = nullptr;      // pinned
  uint32_t d_clock_known = ~0u;     // the value d_clock holds once the queued work ran (~0: unknown)
  bool sort_advances_clock = false; // set while the end_slice sequence is enqueued
  cudaGraphExec_t graph[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};   // [timing][mode]
  size_t restore_smem = 0;
  uint32_t* ws = nullptr;
  uint64_t ws_cap = 0;
  uint32_t* cand = nullptr;
  ReportDev* rep = nullptr;
  ReportDev* rep_sorted = nullptr;
  ReportDev* rep_above = nullptr;
  uint32_t *keys = nullptr, *keys_alt = nullptr, *vals = nullptr, *vals_alt = nullptr;
  uint32_t* bs_buf = nullptr;       // bucket sort: [5][kBsMaxB] bucket arrays + [2][max_candidates]
  uint16_t* export_buf = nullptr;
  // host pinned
  uint32_t* h_counters = nullptr;
  ReportDev* h_rep = nullptr;       // fixed prefix buffer (a CUDA-graph copy target)
  uint64_t h_rep_cap = 0;
  uint32_t sort_bound = 0;          // > 0: the end_slice graph sorts this many slots on the device
  ReportDev* h_big = nullptr;       // larger report copies
  uint64_t h_big_cap = 0;
  // host-buffer scan staging (P:428 double buffering)
  uint32_t* stage[2] = {nullptr, nullptr};
  uint64_t stage_pairs = 0;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_scanned[2] = {nullptr, nullptr};
  cudaEvent_t ev_join = nullptr;
  cudaEvent_t ev_order = nullptr;     // context stream -> caller stream (asse_scan_slice)
  cudaEvent_t ev_scan_last = nullptr; // last scan of this context: scans on any stream are serialised
  // timing
  bool timing = false;
  std::vector<cudaEvent_t> ev_free;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> scan_ev;
  cudaEvent_t ev[12] = {nullptr};
  // last slice
  uint32_t last_n = 0, last_above = 0;
  bool have_reports = false;
  // asse_end_slice_async: one closed slice whose results are still on the way
  bool pending = false;
  uint32_t pend_mode = 0, pend_K = 0;
  cudaEvent_t ev_collect = nullptr;
  // peers
  bool peers = false;
  uint32_t sync_mode = 0, epoch = 0;  // 0 device barrier, 1 caller-ordered, 2 host barrier
  asse_host_barrier_fn host_barrier = nullptr;   // sync_mode 2
  void* host_barrier_arg = nullptr;
  void* peer_touch[kMaxWorld] = {nullptr};
  void* peer_merged[kMaxWorld] = {nullptr};
  void* peer_xchg[kMaxWorld] = {nullptr};
  uint8_t* xchg = nullptr;          // option S: this rank's exchange buffer (count | reports)
  bool begun = false;               // option S, sync_mode 1: end_slice_begin done
  void* peer_signal[kMaxWorld] = {nullptr};
  asse_stats stats{};
  std::string err;
};

#define CK(call)                                                                    \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      c->err = std::string(#call) + ": " + cudaGetErrorString(e_);                  \
      return ASSE_E_CUDA;                                                           \
    }                                                                               \
  } while (0)

#define LAUNCHED(c_) ((c_)->stats.kernel_launches++)

#define NOT_PENDING(c_)                                                                   \
  do {                                                                                    \
    if ((c_)->pending) { (c_)->err = "results of an asynchronous end_slice pending: call " \
                                     "asse_end_slice_wait first"; return ASSE_E_STATE; }   \
  } while (0)


static uint64_t splitmix_next(uint64_t* st) {  // A14
  uint64_t z = (*st += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static uint32_t inv_newton(uint32_t A) {  // A^{-1} mod 2^32 for odd A (A8)
  uint32_t x = A;                           // correct to 3 bits
  for (int it = 0; it < 5; ++it) x *= 2u - A * x;
  return x;
}

static asse_status validate(const asse_config* cfg, std::string* why) {
  auto bad = [&](const char* m) { if (why) *why = m; return ASSE_E_PARAM; };
  if (!cfg) return bad("null config");
  const asse_config& p = *cfg;
  uint32_t kp = p.k_prime ? p.k_prime : p.k;
  if (p.k < 1) return bad("k >= 1");
  if (kp < 1 || kp > p.k) return bad("1 <= k' <= k");
  if (p.k > 16383) return bad("k <= 16383 (15-bit device codes)");
  if (p.r < 2 || p.r > (uint32_t)kMaxR) return bad("2 <= r <= 8");
  if (p.c < 2 || p.u > 16 || p.c + p.u > 32) return bad("c >= 2, u <= 16, c + u <= 32");
  if (p.c + p.u > 24) return bad("device path: c + u <= 24 (32-bit ATV indices)");
  if (p.s < 1 || p.s > p.c) return bad("1 <= s <= c");
  if (!(p.theta > 0)) return bad("theta > 0");
  if (p.g < 128 || p.g > 4096 || (p.g & (p.g - 1))) return bad("device path: g in {128, 256, ..., 4096}");
  if (p.max_candidates < 1) return bad("max_candidates >= 1");
  if (p.world < 1 || p.world > (uint32_t)kMaxWorld || p.rank >= p.world) return bad("rank < world <= 16");
  if (p.frame_shard > 1) return bad("frame_shard is 0 or 1");
  if (p.mangle > 1) return bad("mangle is 0 or 1");
  if (p.frame_shard && ((1u << p.u) % p.world)) return bad("frame_shard: world must divide 2^u frames");
  const uint32_t W = 32 - p.u;
  if (p.c + p.s * (p.r - 1) < W) return bad("completeness: c + s(r-1) >= 32-u (P:324, A10)");
  std::vector<int> cover(W, 0);
  for (uint32_t y = 0; y < p.r; ++y)
    for (uint32_t j = 0; j < p.c; ++j) cover[(p.s * y + j) % W]++;
  bool dup = false;
  for (uint32_t q = 0; q < W; ++q) {
    if (!cover[q]) return bad("completeness: an LBS bit is not covered (P:316)");
    if (cover[q] > 1) dup = true;
  }
  if (!dup) return bad("redundancy: no duplicate position (P:317)");
  return ASSE_OK;
}

static void free_all(Ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->d2h_stream) cudaStreamSynchronize(c->d2h_stream);
  if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
  void* dev[] = {c->pool, c->touch_own, c->active, c->scratch, c->sa_list, c->ws, c->cand, c->rep, c->rep_sorted, c->rep_above, c->keys,
                 c->keys_alt, c->vals, c->vals_alt, c->bs_buf, c->export_buf, c->stage[0],
                 c->stage[1], c->bin_queue, c->bin_sync, c->own_queue, c->own_sync};
  for (void* p : dev) if (p) cudaFree(p);
  if (c->h_counters) cudaFreeHost(c->h_counters);
  if (c->h_clock) cudaFreeHost(c->h_clock);
  if (c->d_clock) cudaFree(c->d_clock);
  for (auto& row : c->graph) for (auto& g : row) if (g) cudaGraphExecDestroy(g);
  if (c->h_rep) cudaFreeHost(c->h_rep);
  if (c->h_big) cudaFreeHost(c->h_big);
  for (int q = 0; q < 2; ++q) {
    if (c->ev_copied[q]) cudaEventDestroy(c->ev_copied[q]);
    if (c->ev_scanned[q]) cudaEventDestroy(c->ev_scanned[q]);
  }
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->ev_order) cudaEventDestroy(c->ev_order);
  if (c->ev_scan_last) cudaEventDestroy(c->ev_scan_last);
  for (auto& pr : c->scan_ev) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
  for (auto e : c->ev_free) cudaEventDestroy(e);
  for (auto e : c->ev) if (e) cudaEventDestroy(e);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->d2h_stream) cudaStreamDestroy(c->d2h_stream);
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  if (c->ev_collect) cudaEventDestroy(c->ev_collect);
  if (c->stream) cudaStreamDestroy(c->stream);
}

template <int CB, int LPAL, int QL = 0>
static cudaError_t fold_occ_t(int* occ) {
  cudaError_t e = cudaFuncSetAttribute(k_fold<CB, LPAL, false, QL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)fold_smem<CB, false>());
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_fold<CB, LPAL, true, QL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)fold_smem<CB, true>());
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, k_fold<CB, LPAL, false, QL>, fold_threads<CB, false>(),
                                                       fold_smem<CB, false>());
}
template <int CB>
static cudaError_t fold_occ_cb(uint32_t lpal, uint32_t ql, int* occ) {
  if (ql == 1) return fold_occ_t<CB, 5, 1>(occ);
  if (ql == 2) return fold_occ_t<CB, 5, 2>(occ);
  if (ql == 3) return fold_occ_t<CB, 5, 3>(occ);
  return lpal == 3 ? fold_occ_t<CB, 3>(occ) : lpal == 4 ? fold_occ_t<CB, 4>(occ) : fold_occ_t<CB, 5>(occ);
}
static cudaError_t fold_occupancy(uint32_t cb, uint32_t lpal, uint32_t ql, int* occ) {
  return cb == 1 ? fold_occ_cb<1>(lpal, ql, occ) : fold_occ_cb<2>(lpal, ql, occ);
}
// fold launch for the geometry: lpal = log2(g/16) capped at 5, ql = log2(g/512) for g > 512
template <int CB, bool WEIGH = false>
static void launch_fold(uint32_t lpal, uint32_t ql, unsigned blocks, cudaStream_t s, const FoldParams& fp) {
  const size_t sm = fold_smem<CB, WEIGH>();
  const int th = fold_threads<CB, WEIGH>();
  if (ql == 1) k_fold<CB, 5, WEIGH, 1><<<blocks, th, sm, s>>>(fp);
  else if (ql == 2) k_fold<CB, 5, WEIGH, 2><<<blocks, th, sm, s>>>(fp);
  else if (ql == 3) k_fold<CB, 5, WEIGH, 3><<<blocks, th, sm, s>>>(fp);
  else if (lpal == 3) k_fold<CB, 3, WEIGH><<<blocks, th, sm, s>>>(fp);
  else if (lpal == 4) k_fold<CB, 4, WEIGH><<<blocks, th, sm, s>>>(fp);
  else k_fold<CB, 5, WEIGH><<<blocks, th, sm, s>>>(fp);
}

// Launch with programmatic stream serialization (PDL): the kernel may start while the
// previous kernel in the stream drains; it waits with griddepcontrol.wait.
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Binned scan (asse_scan_bin.cuh): cooperative launch (every CTA co-resident: they wait
// on each other's rounds). Binned scans of every context in the process are serialized
// on one event so that two such grids never share the GPU.
static cudaEvent_t g_bin_last[64] = {nullptr};

template <int CB, bool MP, int RR>
static cudaError_t coop_launch_bin(Ctx* c, const uint2* pk, uint64_t n, const BinScanParams& bp, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(c->bin_G);
  cfg.blockDim = dim3(kBinThreads);
  cfg.dynamicSmemBytes = c->bin_smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_scan_bin<CB, MP, RR>, pk, n, bp);
}
template <int CB, bool MP>
static cudaError_t coop_launch_bin_rr(Ctx* c, const uint2* pk, uint64_t n, const BinScanParams& bp, cudaStream_t st) {
  if (c->bin_rr == 0) return coop_launch_bin<CB, MP, 0>(c, pk, n, bp, st);
  if (c->bin_rr == 1) return coop_launch_bin<CB, MP, 1>(c, pk, n, bp, st);
  return coop_launch_bin<CB, MP, 2>(c, pk, n, bp, st);
}

static asse_status launch_scan_bin(Ctx* c, const uint2* pk, uint64_t n, const ScanParams& sp, cudaStream_t st) {
  const uint32_t G = c->bin_G;
  if (!c->bin_queue) {
    CK(cudaMalloc(&c->bin_queue, (size_t)kBinNB * G * kBinQG * kBinQCap * 4));
    CK(cudaMalloc(&c->bin_sync, (2 * kBinNB + (size_t)kBinNB * G * kBinQG) * kBinPad * 4));
  }
  const int dev = c->device & 63;
  if (!g_bin_last[dev]) CK(cudaEventCreateWithFlags(&g_bin_last[dev], cudaEventDisableTiming));
  CK(cudaStreamWaitEvent(st, g_bin_last[dev], 0));
  BinScanParams bp{};
  bp.sp = sp;
  bp.queue = c->bin_queue;
  bp.qcnt = c->bin_sync + 2 * kBinNB * kBinPad;
  bp.sync = c->bin_sync;
  const uint64_t row_words = (uint64_t)c->F * c->E * c->wpa;
  bp.base_word = (uint32_t)(c->bin_rr * row_words);
  bp.total_words = c->n_atv_full * c->wpa - bp.base_word;
  // empirical (B200, C3-C5 traffic): calls of 40-127 full rounds run faster with 3/4 tiles
  // (C3, 66 rounds: 0.333 ms at 1536 packets per round vs 0.351 at 2048), shorter and
  // longer calls with full tiles (C4, 33 rounds: 0.161 vs 0.178; C5, 330 rounds)
  bp.tile_bytes = c->bin_tile;
  const uint64_t full_rounds = n / ((uint64_t)G * (c->bin_tile / 8));
  if (!getenv("ASSE_SCAN_TILE") && full_rounds >= 40 && full_rounds < 128 && c->bin_tile >= 16384)
    bp.tile_bytes = c->bin_tile / 4 * 3;
  bp.inv = c->bin_inv;
  bp.wpo = c->bin_wpo;
  static const bool prof = getenv("ASSE_SCAN_PROF") != nullptr;
  if (prof) {
    static unsigned long long* dprof = nullptr;
    if (!dprof) CK(cudaMalloc(&dprof, 16 * 1024 * 8));
    bp.prof = dprof;
  }
  CK(cudaMemsetAsync(c->bin_sync, 0, (2 * kBinNB + (size_t)kBinNB * G * kBinQG) * kBinPad * 4, st));
  cudaError_t e;
  if (c->cfg.mangle) e = c->cb == 1 ? coop_launch_bin_rr<1, true>(c, pk, n, bp, st) : coop_launch_bin_rr<2, true>(c, pk, n, bp, st);
  else e = c->cb == 1 ? coop_launch_bin_rr<1, false>(c, pk, n, bp, st) : coop_launch_bin_rr<2, false>(c, pk, n, bp, st);
  if (e == cudaErrorCooperativeLaunchTooLarge) {
    // fewer SMs than at init (e.g. shared with another context): k_scan does this call
    cudaGetLastError();
    return ASSE_E_CAPACITY;
  }
  CK(e);
  CK(cudaEventRecord(g_bin_last[dev], st));
  if (bp.prof) {   // tools: ASSE_SCAN_PROF=1 prints per-phase cycles of the binned scan (syncs)
    std::vector<unsigned long long> h((size_t)G * 16);
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(h.data(), bp.prof, h.size() * 8, cudaMemcpyDeviceToHost));
    const char* nm[13] = {"b_bin", "b_wait_reserve", "b_copy", "-", "-", "-",
                          "-", "-", "-", "c0_wait", "c0_drain", "c1_wait", "c1_drain"};
    fprintf(stderr, "k_scan_bin n=%llu G=%u:", (unsigned long long)n, G);
    for (int q = 0; q < 13; ++q) {
      double sum = 0, mx = 0;
      for (uint32_t b = 0; b < G; ++b) { sum += (double)h[b * 16 + q]; mx = std::max(mx, (double)h[b * 16 + q]); }
      fprintf(stderr, " %s %.0f/%.0f;", nm[q], sum / G, mx);
    }
    fprintf(stderr, "\n");
  }
  c->stats.scan_bin_launches++;
  return ASSE_OK;
}

template <int CB, bool MP, class Geo>
static cudaError_t coop_launch_own(Ctx* c, const uint2* pk, uint64_t n, const OwnScanParams& op, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  // tools only: ASSE_OWN_GRID = CTAs of the packet-owned scan (>= owners; default one per SM)
  static const uint32_t grid_env = getenv("ASSE_OWN_GRID") ? (uint32_t)atoi(getenv("ASSE_OWN_GRID")) : 0u;
  cfg.gridDim = dim3(grid_env >= c->own_O && grid_env <= c->bin_G ? grid_env : c->bin_G);
  cfg.blockDim = dim3(kOwnThreads);
  cfg.dynamicSmemBytes = c->own_smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_scan_own<CB, MP, Geo>, pk, n, op);
}

static asse_status launch_scan_own(Ctx* c, const uint2* pk, uint64_t n, const ScanParams& sp, cudaStream_t st) {
  const uint32_t G = c->bin_G, O = c->own_O;
  const size_t sync_words = (2 * kOwnNB + (size_t)kOwnNB * O * kOwnQG) * kBinPad;
  if (!c->own_queue) {
    CK(cudaMalloc(&c->own_queue, (size_t)kOwnNB * O * kOwnQG * kOwnQCap * sizeof(uint2)));
    CK(cudaMalloc(&c->own_sync, 2 * sync_words * 4));
    CK(cudaMemsetAsync(c->own_sync, 0, 2 * sync_words * 4, st));
  }
  const int dev = c->device & 63;
  if (!g_bin_last[dev]) CK(cudaEventCreateWithFlags(&g_bin_last[dev], cudaEventDisableTiming));
  CK(cudaStreamWaitEvent(st, g_bin_last[dev], 0));
  OwnScanParams op{};
  op.sp = sp;
  op.queue = c->own_queue;
  // this launch's counters are zero (set at allocation or by the previous launch); the
  // kernel zeroes the other set for the next launch (scans of a device are serialised)
  uint32_t* cur = c->own_sync + (size_t)c->own_parity * sync_words;
  op.qcnt = cur + 2 * kOwnNB * kBinPad;
  op.sync = cur;
  op.sync_next = c->own_sync + (size_t)(c->own_parity ^ 1u) * sync_words;
  op.sync_words = (uint32_t)sync_words;
  op.O = O;
  op.lg_ngrp = c->own_lg_ngrp;
  op.lg_wg = c->own_lg_wg;
  op.tile_bytes = c->own_tile;
  static const bool prof = getenv("ASSE_SCAN_PROF") != nullptr;
  if (prof) {
    static unsigned long long* dprof = nullptr;
    if (!dprof) CK(cudaMalloc(&dprof, 16 * 1024 * 8));
    op.prof = dprof;
  }
  cudaError_t e;
  const asse_config& g = c->cfg;
  const bool c3 = g.u == 4 && g.c == 12 && g.s == 6 && g.g == 512 && g.r == 4 && c->own_lg_ngrp == 3 && c->own_lg_wg == 1 &&
                  !getenv("ASSE_SCAN_OWN_GENERIC");   // the BASELINE C3-C5 geometry: constants folded
  if (c3) {
    if (g.mangle) e = c->cb == 1 ? coop_launch_own<1, true, GeoC3>(c, pk, n, op, st) : coop_launch_own<2, true, GeoC3>(c, pk, n, op, st);
    else e = c->cb == 1 ? coop_launch_own<1, false, GeoC3>(c, pk, n, op, st) : coop_launch_own<2, false, GeoC3>(c, pk, n, op, st);
  } else {
    if (g.mangle) e = c->cb == 1 ? coop_launch_own<1, true, GeoRt>(c, pk, n, op, st) : coop_launch_own<2, true, GeoRt>(c, pk, n, op, st);
    else e = c->cb == 1 ? coop_launch_own<1, false, GeoRt>(c, pk, n, op, st) : coop_launch_own<2, false, GeoRt>(c, pk, n, op, st);
  }
  if (e == cudaErrorCooperativeLaunchTooLarge) {
    cudaGetLastError();
    return ASSE_E_CAPACITY;
  }
  CK(e);
  c->own_parity ^= 1u;                           // launched: the next call uses the set it zeroes
  CK(cudaEventRecord(g_bin_last[dev], st));
  if (op.prof) {
    std::vector<unsigned long long> h((size_t)G * 16);
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(h.data(), op.prof, h.size() * 8, cudaMemcpyDeviceToHost));
    const char* nm[13] = {"b_bin", "b_wait_reserve", "b_copy", "b_bin_wait_tile", "t_start", "t_shipped",
                          "t_drained", "-", "-", "c0_wait", "c0_drain", "c1_wait", "c1_drain"};
    {   // timeline (globaltimer ns) relative to the earliest CTA start
      unsigned long long t0 = ~0ull;
      for (uint32_t b = 0; b < G; ++b) t0 = std::min(t0, h[b * 16 + 4]);
      for (int q = 4; q <= 6; ++q) {
        unsigned long long mn = ~0ull, mx = 0;
        for (uint32_t b = 0; b < G; ++b) {
          if (q == 6 || b < G) { mn = std::min(mn, h[b * 16 + q] - t0); mx = std::max(mx, h[b * 16 + q] - t0); }
        }
        fprintf(stderr, "k_scan_own timeline %s: min %.1f us max %.1f us\n", nm[q], mn / 1e3, mx / 1e3);
      }
    }
    fprintf(stderr, "k_scan_own n=%llu G=%u O=%u:", (unsigned long long)n, G, O);
    for (int q = 0; q < 13; ++q) {
      double sum = 0, mx = 0;
      for (uint32_t b = 0; b < G; ++b) { sum += (double)h[b * 16 + q]; mx = std::max(mx, (double)h[b * 16 + q]); }
      fprintf(stderr, " %s %.0f/%.0f;", nm[q], sum / G, mx);
    }
    fprintf(stderr, "\n");
  }
  c->stats.scan_own_launches++;
  return ASSE_OK;
}

static asse_status launch_scan(Ctx* c, const uint32_t* d_pairs, uint64_t n, cudaStream_t st) {
  if (n == 0) return ASSE_OK;
  ScanParams p{};
  p.touch = c->touch;
  p.kbh = c->K_bh;
  p.A = c->A;
  p.g = c->cfg.g; p.r = c->cfg.r; p.u = c->cfg.u; p.c = c->cfg.c; p.W = c->W;
  p.fmask = (1u << c->cfg.u) - 1u;
  p.cmask = (1u << c->cfg.c) - 1u;
  p.wpa = c->wpa;
  for (int y = 0; y < kMaxR; ++y) p.shift[y] = c->shift[y];
  const uint64_t tiles = ((n / 2) * 16 + kScanTileBytes - 1) / kScanTileBytes;   // 16 KB tiles
  const uint64_t blocks = std::max<uint64_t>(1, std::min<uint64_t>(tiles, (uint64_t)c->scan_grid));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->timing) {
    if (c->ev_free.size() < 2) {
      for (int q = 0; q < 8; ++q) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        c->ev_free.push_back(e);
      }
    }
    e0 = c->ev_free.back(); c->ev_free.pop_back();
    e1 = c->ev_free.back(); c->ev_free.pop_back();
    CK(cudaEventRecord(e0, st));
  }
  const uint2* pk = reinterpret_cast<const uint2*>(d_pairs);
  // every scan of this context waits for the previous one, whatever stream either runs on:
  // the owner write-backs of k_scan_bin / k_scan_own read-OR-write touch words, which a
  // concurrent k_scan's REDs into the same bitmap could otherwise interleave with
  CK(cudaStreamWaitEvent(st, c->ev_scan_last, 0));
  const bool use_own = c->own_ok && (c->scan_variant == 3 ||
                                     (c->scan_variant == 0 && tiles * kScanTileBytes >= (uint64_t)c->bin_G * kOwnMinTilesPerCta * c->own_tile));
  const bool use_bin = !use_own && c->bin_ok && (c->scan_variant == 2 ||
                                     (c->scan_variant == 0 && tiles * kScanTileBytes >= (uint64_t)c->bin_G * kBinMinTilesPerCta * c->bin_tile));
  asse_status bs = use_own ? launch_scan_own(c, pk, n, p, st) : use_bin ? launch_scan_bin(c, pk, n, p, st) : ASSE_E_CAPACITY;
  if ((use_own || use_bin) && bs != ASSE_OK && bs != ASSE_E_CAPACITY) return bs;
  if ((use_own || use_bin) && bs == ASSE_OK) {
  } else if (c->cfg.mangle) {
    if (c->cb == 1) k_scan<1, true><<<(unsigned)blocks, kScanThreads, kScanSmem, st>>>(pk, n, p);
    else k_scan<2, true><<<(unsigned)blocks, kScanThreads, kScanSmem, st>>>(pk, n, p);
  } else {
    if (c->cb == 1) k_scan<1><<<(unsigned)blocks, kScanThreads, kScanSmem, st>>>(pk, n, p);
    else k_scan<2><<<(unsigned)blocks, kScanThreads, kScanSmem, st>>>(pk, n, p);
  }
  CK(cudaGetLastError());
  CK(cudaEventRecord(c->ev_scan_last, st));
  LAUNCHED(c);
  c->stats.scan_launches++;
  c->stats.packets_scanned += n;
  if (c->timing) {
    CK(cudaEventRecord(e1, st));
    c->scan_ev.emplace_back(e0, e1);
  }
  return ASSE_OK;
}

static asse_status harvest_scan_timing(Ctx* c) {
  for (auto& pr : c->scan_ev) {
    float ms = 0;
    CK(cudaEventSynchronize(pr.second));
    CK(cudaEventElapsedTime(&ms, pr.first, pr.second));
    c->stats.scan_ms_total += ms;
    c->ev_free.push_back(pr.first);
    c->ev_free.push_back(pr.second);
  }
  c->scan_ev.clear();
  return ASSE_OK;
}

static asse_status do_merge(Ctx* c) {
  if (!c->peers) return ASSE_OK;
  if (c->shard) {
    MergeShardParams mp{};
    for (uint32_t w = 0; w < c->cfg.world; ++w) mp.touch[w] = reinterpret_cast<const uint4*>(c->peer_touch[w]);
    mp.merged = reinterpret_cast<uint4*>(c->merged);
    mp.world = c->cfg.world;
    const uint64_t frame4 = (uint64_t)c->E * c->wpa / 4;     // uint4 words per (row, frame) slab
    mp.row_local = frame4 * c->Fl;
    mp.row_global = frame4 * c->F;
    mp.frame_off = frame4 * c->z_base;
    mp.n = mp.row_local * c->cfg.r;
    const uint64_t blocks = std::min<uint64_t>((mp.n + 255) / 256, (uint64_t)c->sms * 4);
    k_merge_shard<<<(unsigned)blocks, 256, 0, c->stream>>>(mp);
    CK(cudaGetLastError());
    LAUNCHED(c);
    return ASSE_OK;
  }
  MergeParams mp{};
  for (uint32_t w = 0; w < c->cfg.world; ++w) {
    mp.touch[w] = reinterpret_cast<const uint4*>(c->peer_touch[w]);
    mp.merged[w] = reinterpret_cast<uint4*>(c->peer_merged[w]);
  }
  mp.world = c->cfg.world;
  const uint64_t n4 = c->n_atv_full * c->wpa / 4;
  const uint64_t per = (n4 + c->cfg.world - 1) / c->cfg.world;
  mp.lo = per * c->cfg.rank;
  mp.hi = std::min<uint64_t>(n4, mp.lo + per);
  if (mp.lo >= mp.hi) return ASSE_OK;
  uint64_t blocks = std::min<uint64_t>((mp.hi - mp.lo + 255) / 256, (uint64_t)c->sms * 4);
  k_merge_or<<<(unsigned)blocks, 256, 0, c->stream>>>(mp);
  CK(cudaGetLastError());
  LAUNCHED(c);
  return ASSE_OK;
}

// Cross-rank barrier of the eager end_slice (sync_mode 0: stream-ordered device barrier
// over the peer signal pads; sync_mode 2: this rank's queued work completes, then the
// caller's host barrier — no kernel ever waits for another rank's kernel).
static asse_status device_barrier(Ctx* c);
static asse_status rank_barrier(Ctx* c) {
  if (c->sync_mode == 0) return device_barrier(c);
  CK(cudaStreamSynchronize(c->stream));
  if (!c->host_barrier) { c->err = "sync_mode 2 without asse_set_host_barrier"; return ASSE_E_PEER; }
  if (c->host_barrier(c->host_barrier_arg) != 0) { c->err = "host barrier callback failed"; return ASSE_E_PEER; }
  c->stats.host_barriers++;
  return ASSE_OK;
}

static asse_status device_barrier(Ctx* c) {
  BarrierParams bp{};
  for (uint32_t w = 0; w < c->cfg.world; ++w) bp.pads[w] = reinterpret_cast<uint32_t*>(c->peer_signal[w]);
  bp.world = c->cfg.world;
  bp.rank = c->cfg.rank;
  bp.epoch = ++c->epoch;
  k_barrier<<<1, 32, 0, c->stream>>>(bp);
  CK(cudaGetLastError());
  LAUNCHED(c);
  return ASSE_OK;
}

}  // namespace

extern "C" {

asse_status asse_validate(const asse_config* cfg, char* why, size_t n) {
  std::string w;
  asse_status st = validate(cfg, &w);
  if (why && n) snprintf(why, n, "%s", st == ASSE_OK ? "" : w.c_str());
  return st;
}

const char* asse_last_error(const void* ctx) {
  if (!ctx) return "no context";
  return static_cast<const Ctx*>(ctx)->err.c_str();
}

asse_status asse_init(const asse_config* cfg, void** out) {
  if (!out) return ASSE_E_PARAM;
  *out = nullptr;
  std::string why;
  if (validate(cfg, &why) != ASSE_OK) {
    fprintf(stderr, "asse_init: %s\n", why.c_str());
    return ASSE_E_PARAM;
  }
  Ctx* c = new Ctx();
  c->cfg = *cfg;
  const asse_config& p = c->cfg;
  c->F = 1u << p.u;
  c->E = 1u << p.c;
  c->W = 32 - p.u;
  c->two_k = 2 * p.k;
  c->kp = p.k_prime ? p.k_prime : p.k;
  c->a = p.g / c->two_k;                        // P:256, A7
  c->b = p.g - c->a * (c->two_k - 1);
  c->cb = (c->two_k <= 126) ? 1 : 2;           // A2
  c->wpa = p.g / 32;
  c->lpa_log2 = (p.g == 128) ? 3 : (p.g == 256 ? 4 : 5);
  c->q_log2 = (p.g <= 512) ? 0 : (p.g == 1024 ? 1 : (p.g == 2048 ? 2 : 3));
  for (uint32_t y = 0; y < p.r; ++y) c->shift[y] = (p.s * y) % c->W;
  c->shard = p.frame_shard && p.world > 1;
  c->Fl = c->shard ? c->F / p.world : c->F;
  c->z_base = c->shard ? p.rank * c->Fl : 0;
  c->n_atv_full = (uint64_t)p.r * c->F * c->E;
  c->n_atv = (uint64_t)p.r * c->Fl * c->E;
  c->n_at = c->n_atv * p.g;
  // W_theta = ceil(g - g e^{-theta/g}) (A15)
  double wt = (double)p.g - (double)p.g * exp(-p.theta / (double)p.g);
  double wc = ceil(wt);
  c->w_theta = (wc > (double)p.g) ? p.g + 1 : (uint32_t)wc;
  uint64_t st = p.seed;
  if (!p.mangle) {
    c->A = (uint32_t)(splitmix_next(&st) >> 32) | 1u;
    c->K_bh = splitmix_next(&st);
    c->A_inv = inv_newton((uint32_t)c->A);
  } else {                                    // A in [1, p-1]; A^{-1} = A^{p-2} (Fermat)
    c->A = splitmix_next(&st) % (kMangleP - 1) + 1;
    c->K_bh = splitmix_next(&st);
    uint64_t r = 1, b = c->A;
    for (uint64_t e = kMangleP - 2; e; e >>= 1) {
      if (e & 1) r = mulmod_p(r, b);
      b = mulmod_p(b, b);
    }
    c->A_inv = r;
  }
  c->device = p.device;
  c->stats.w_theta = c->w_theta;
  c->stats.code_bytes = c->cb;
  auto fail = [&](asse_status s) {
    fprintf(stderr, "asse_init: %s\n", c->err.c_str());
    free_all(c);
    delete c;
    return s;
  };
#define CKI(call)                                                       \
  do {                                                                  \
    cudaError_t e_ = (call);                                            \
    if (e_ != cudaSuccess) {                                            \
      c->err = std::string(#call) + ": " + cudaGetErrorString(e_);      \
      return fail(ASSE_E_CUDA);                                         \
    }                                                                   \
  } while (0)
  CKI(cudaSetDevice(c->device));
  CKI(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->device));
  CKI(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  {
    int occ = 0;
    CKI(cudaFuncSetAttribute(k_scan<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kScanSmem));
    CKI(cudaFuncSetAttribute(k_scan<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kScanSmem));
    CKI(cudaFuncSetAttribute(k_scan<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kScanSmem));
    CKI(cudaFuncSetAttribute(k_scan<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kScanSmem));
    if (c->cb == 1) CKI(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_scan<1>, kScanThreads, kScanSmem));
    else CKI(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_scan<2>, kScanThreads, kScanSmem));
    c->scan_grid = std::max(1, occ) * c->sms;
    {
      // binned scan: words per owner (multiple of 4) must fit next to the ring and bins
      int optin = 0, coop = 0;
      CKI(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
      CKI(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, c->device));
      // rows below bin_rr take the direct RED route, the rest are binned (ASSE_SCAN_RR
      // overrides, tools only); 4096 binned updates per CTA per round
      if (const char* e = getenv("ASSE_SCAN_RR")) c->bin_rr = (uint32_t)std::min(2, std::max(0, atoi(e)));
      const uint64_t row_words = (uint64_t)c->F * c->E * c->wpa;
      c->bin_G = (uint32_t)c->sms;
      // small geometries (whole bitmap <= 64 KiB per SM) bin every row (measured: C2 0.097 ms
      // at RR = 0 vs 0.121 at RR = 1; C3-C5 are fastest at RR = 1)
      if (!getenv("ASSE_SCAN_RR") && (p.r * row_words) / c->bin_G <= 16384) c->bin_rr = 0;
      if (((p.r - c->bin_rr) * row_words) / c->bin_G <= 256) c->bin_rr = 0;
      const uint64_t words = (p.r - c->bin_rr) * row_words;
      // packets per CTA per round: a multiple of 1024 (every binning thread handles the same
      // number of 16-B groups), ~kBinCap * 64 binned updates per round (tools: ASSE_SCAN_TILE)
      {
        uint32_t pk = ((uint32_t)(kBinCap * 64) / (4 - c->bin_rr) + 512) / 1024 * 1024;
        if (const char* e = getenv("ASSE_SCAN_TILE")) pk = ((uint32_t)atoi(e) + 1u) & ~1u;
        c->bin_tile = std::max<uint32_t>(1024, pk) * 8;
      }
      c->bin_wpo = (uint32_t)(((words + c->bin_G - 1) / c->bin_G + 3) & ~3ull);
      c->bin_inv = (uint32_t)std::min<uint64_t>(0xFFFFFFFFull, ((1ull << 40) + c->bin_wpo - 1) / c->bin_wpo);
      c->bin_smem = bin_smem_bytes(c->bin_G, c->bin_wpo, c->bin_tile);
      c->bin_ok = coop && p.r == 4 && c->bin_wpo > 256 && (uint64_t)((c->bin_G + kBinQG - 1) / kBinQG) * kBinCap <= kBinQCap &&
                  (uint32_t)c->bin_G <= kMaxOwners && words < (1ull << 25) && c->bin_wpo < (1u << 27) &&
                  c->bin_smem + 2048 <= (size_t)optin;
      if (c->bin_ok) {
        void* fns[12] = {(void*)k_scan_bin<1, false, 0>, (void*)k_scan_bin<2, false, 0>, (void*)k_scan_bin<1, true, 0>,
                         (void*)k_scan_bin<2, true, 0>, (void*)k_scan_bin<1, false, 1>, (void*)k_scan_bin<2, false, 1>,
                         (void*)k_scan_bin<1, true, 1>, (void*)k_scan_bin<2, true, 1>, (void*)k_scan_bin<1, false, 2>,
                         (void*)k_scan_bin<2, false, 2>, (void*)k_scan_bin<1, true, 2>, (void*)k_scan_bin<2, true, 2>};
        for (void* f : fns) CKI(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->bin_smem));
        int bocc = 0;
        CKI(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bocc, k_scan_bin<1, false, 2>, kBinThreads, c->bin_smem));
        c->bin_ok = bocc >= 1;
      }
      c->stats.scan_rows_red = c->bin_rr;
      c->stats.scan_bin_ok = c->bin_ok ? 1u : 0u;
      // packet-owned scan: O = F * NGRP owners (NGRP word groups per ATV, a power of two
      // dividing g/32, F * NGRP <= SMs), slice = r x 2^c ATVs x WG words in shared memory
      {
        const uint32_t F = 1u << p.u;
        uint32_t lg_wpa = 0;
        while ((1u << lg_wpa) < c->wpa) ++lg_wpa;
        uint32_t lg_ngrp = 0;
        while (lg_ngrp < lg_wpa && (F << (lg_ngrp + 1)) <= (uint32_t)c->sms) ++lg_ngrp;
        c->own_lg_ngrp = lg_ngrp;
        c->own_lg_wg = lg_wpa - lg_ngrp;
        c->own_O = F << lg_ngrp;
        // ~16 entries per bin per round on average (CAP = 30): 2048 packets at O = 128
        c->own_tile = std::min<uint32_t>(2048u, std::max<uint32_t>(1024u, c->own_O * 16u) / 1024u * 1024u) * 8u;
        if (const char* e = getenv("ASSE_SCAN_TILE")) c->own_tile = ((uint32_t)atoi(e) + 255u) / 256u * 256u * 8u;
        const uint64_t slice_words = (uint64_t)p.r << (p.c + c->own_lg_wg);
        c->own_smem = own_smem_bytes(c->own_O, (uint32_t)std::min<uint64_t>(slice_words, 1u << 30), c->own_tile);
        c->own_ok = coop && p.r == 4 && (1u << lg_wpa) == c->wpa && c->own_O <= (uint32_t)c->sms && c->own_lg_wg <= p.u &&
                    c->own_O <= kOwnMaxOwners && c->own_O >= 2 &&
                    (uint64_t)((c->sms + kOwnQG - 1) / kOwnQG) * kOwnCap <= kOwnQCap &&
                    slice_words <= (1u << 20) && c->own_smem + 2048 <= (size_t)optin &&
                    !getenv("ASSE_SCAN_NO_OWN");
        if (c->own_ok) {
          void* fns[8] = {(void*)k_scan_own<1, false, GeoRt>, (void*)k_scan_own<2, false, GeoRt>,
                          (void*)k_scan_own<1, true, GeoRt>, (void*)k_scan_own<2, true, GeoRt>,
                          (void*)k_scan_own<1, false, GeoC3>, (void*)k_scan_own<2, false, GeoC3>,
                          (void*)k_scan_own<1, true, GeoC3>, (void*)k_scan_own<2, true, GeoC3>};
          for (void* f : fns) CKI(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->own_smem));
          int oocc = 0;
          CKI(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oocc, k_scan_own<1, false, GeoRt>, kOwnThreads, c->own_smem));
          c->own_ok = oocc >= 1;
        }
        c->stats.scan_own_ok = c->own_ok ? 1u : 0u;
      }
    }
    CKI(fold_occupancy(c->cb, c->lpa_log2, c->q_log2, &occ));
    c->fold_grid = std::max(1, occ) * c->sms;
  }
  CKI(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  CKI(cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking));
  CKI(cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming));
  CKI(cudaEventCreateWithFlags(&c->ev_collect, cudaEventDisableTiming));
  const uint64_t bm_bytes = c->n_atv * c->wpa * 4;            // local (active, merged)
  const uint64_t touch_bytes = c->n_atv_full * c->wpa * 4;     // whole geometry
  CKI(cudaMalloc(&c->pool, c->n_at * c->cb));
  CKI(cudaMalloc(&c->touch_own, touch_bytes));
  CKI(cudaMalloc(&c->active, bm_bytes));
  {
    const size_t aat_b = (size_t)p.r * c->Fl * 8, cnt_b = ((size_t)p.r * c->Fl * 4 + 255) & ~(size_t)255;
    const size_t bits_b = (size_t)p.r * c->Fl * ((c->E + 31) / 32) * 4;
    c->scratch_bytes = aat_b + cnt_b + 256 + bits_b;
    CKI(cudaMalloc(&c->scratch, c->scratch_bytes));
    uint8_t* b0 = (uint8_t*)c->scratch;
    c->aat = (unsigned long long*)b0;
    c->sa_cnt = (uint32_t*)(b0 + aat_b);
    c->counters = (uint32_t*)(b0 + aat_b + cnt_b);
    c->sa_bits = (uint32_t*)(b0 + aat_b + cnt_b + 256);
  }
  CKI(cudaMalloc(&c->sa_list, (size_t)p.r * c->Fl * c->E * 4));
  {
    // restore geometry (Alg. 4 join plan), parts CTAs per frame
    RestoreParams& rp = c->rp0;
    rp.max_cand = p.max_candidates;
    rp.r = p.r; rp.u = p.u; rp.c = p.c; rp.W = c->W; rp.F = c->Fl;
    rp.z_base = c->z_base;
    rp.sys_fence = c->shard ? 1u : 0u;
    rp.A_inv = c->A_inv; rp.mangle_p = p.mangle; rp.g = p.g; rp.wpa = c->wpa; rp.theta = p.theta;
    rp.cells = (double)p.g * (double)c->E;
    rp.parts = (uint32_t)std::max<int>(1, std::min<int>(16, (2 * c->sms) / (int)c->Fl));
    std::vector<uint8_t> known(c->W, 0);
    for (uint32_t y = 0; y < p.r; ++y) {
      rp.shift[y] = c->shift[y];
      uint32_t ov = 0, nf = 0;
      for (uint32_t j = 0; j < p.c; ++j) {
        uint32_t pos = (c->shift[y] + j) % c->W;
        if (known[pos]) ov |= 1u << j;
        else rp.freepos[y][nf++] = (uint8_t)j;
      }
      for (uint32_t j = 0; j < p.c; ++j) known[(c->shift[y] + j) % c->W] = 1;
      rp.ov[y] = ov;
      rp.nfree[y] = nf;
      {   // free positions (ascending) as at most two contiguous runs
        uint32_t n1 = 0;
        while (n1 < nf && rp.freepos[y][n1] == rp.freepos[y][0] + n1) ++n1;
        uint32_t n2 = 0;
        while (n1 + n2 < nf && rp.freepos[y][n1 + n2] == rp.freepos[y][n1] + n2) ++n2;
        if (n1 + n2 != nf) {   // unreachable for an admissible geometry (window = cyclic interval)
          c->err = "restore plan: the free positions of a row are not two runs";
          return fail(ASSE_E_PARAM);
        }
        rp.dep_n1[y] = (uint8_t)n1;
        rp.dep_sh1[y] = nf ? rp.freepos[y][0] : 0;
        rp.dep_sh2[y] = (n1 < nf) ? (uint8_t)(rp.freepos[y][n1] - n1) : 0;
      }
      rp.use_enum_max[y] = (nf <= 20) ? 4u : 0u;
    }
    c->restore_smem = (size_t)p.r * ((c->E + 31) / 32) * 4;
    if (c->restore_smem > 48 * 1024)
      CKI(cudaFuncSetAttribute(k_restore, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->restore_smem));
    c->ws_cap = 1u << 16;   // partial LBS per CTA and join level
    CKI(cudaMalloc(&c->ws, (size_t)c->Fl * rp.parts * 2 * c->ws_cap * 4));
  }
  CKI(cudaMalloc(&c->cand, (size_t)p.max_candidates * 4));
  CKI(cudaMalloc(&c->rep, (size_t)p.max_candidates * sizeof(ReportDev)));
  CKI(cudaMalloc(&c->rep_sorted, (size_t)p.max_candidates * sizeof(ReportDev)));
  CKI(cudaMalloc(&c->rep_above, (size_t)p.max_candidates * sizeof(ReportDev)));
  CKI(cudaMalloc(&c->keys, (size_t)p.max_candidates * 4));
  CKI(cudaMalloc(&c->keys_alt, (size_t)p.max_candidates * 4));
  CKI(cudaMalloc(&c->vals, (size_t)p.max_candidates * 4));
  CKI(cudaMalloc(&c->vals_alt, (size_t)p.max_candidates * 4));
  CKI(cudaMalloc(&c->bs_buf, (5ull * kBsMaxB + 2ull * p.max_candidates) * 4));
  CKI(cudaMallocHost(&c->h_counters, 64));
  CKI(cudaMallocHost(&c->h_clock, 64));
  CKI(cudaMalloc(&c->d_clock, 64));
  c->h_rep_cap = 4096;   // reports fetched together with the counters (one sync)
  CKI(cudaMallocHost(&c->h_rep, c->h_rep_cap * sizeof(ReportDev)));
  for (auto& e : c->ev) CKI(cudaEventCreate(&e));
  for (int q = 0; q < 2; ++q) {
    CKI(cudaEventCreateWithFlags(&c->ev_copied[q], cudaEventDisableTiming));
    CKI(cudaEventCreateWithFlags(&c->ev_scanned[q], cudaEventDisableTiming));
  }
  CKI(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  CKI(cudaEventCreateWithFlags(&c->ev_order, cudaEventDisableTiming));
  CKI(cudaEventCreateWithFlags(&c->ev_scan_last, cudaEventDisableTiming));
  CKI(cudaEventRecord(c->ev_scan_last, c->stream));
  // InitAT: every AT = 2k
  {
    uint64_t blocks = std::min<uint64_t>((c->n_at + 255) / 256, (uint64_t)c->sms * 16);
    if (c->cb == 1) k_fill_u8<<<(unsigned)blocks, 256, 0, c->stream>>>((uint8_t*)c->pool, (uint8_t)c->two_k, c->n_at);
    else k_fill_u16<<<(unsigned)blocks, 256, 0, c->stream>>>((uint16_t*)c->pool, (uint16_t)c->two_k, c->n_at);
    CKI(cudaGetLastError());
    LAUNCHED(c);
  }
  CKI(cudaMemsetAsync(c->touch_own, 0, touch_bytes, c->stream));
  CKI(cudaMemsetAsync(c->active, 0, bm_bytes, c->stream));
  CKI(cudaStreamSynchronize(c->stream));
  c->touch = c->touch_own;
  c->C0 = 0;
  c->t = 0;
#undef CKI
  *out = c;
  return ASSE_OK;
}

void asse_destroy(void* ctx) {
  if (!ctx) return;
  Ctx* c = static_cast<Ctx*>(ctx);
  free_all(c);
  delete c;
}

asse_status asse_set_timing(void* ctx, int enable) {
  if (!ctx) return ASSE_E_PARAM;
  static_cast<Ctx*>(ctx)->timing = enable != 0;
  return ASSE_OK;
}

asse_status asse_set_scan_variant(void* ctx, int variant) {
  if (!ctx) return ASSE_E_PARAM;
  Ctx* c = static_cast<Ctx*>(ctx);
  if (variant < 0 || variant > 3) {
    c->err = "scan variant is 0 (auto), 1 (direct), 2 (binned) or 3 (packet-owned)";
    return ASSE_E_PARAM;
  }
  if (variant == 2 && !c->bin_ok) { c->err = "binned scan unavailable for this geometry/device"; return ASSE_E_PARAM; }
  if (variant == 3 && !c->own_ok) { c->err = "packet-owned scan unavailable for this geometry/device"; return ASSE_E_PARAM; }
  c->scan_variant = variant;
  return ASSE_OK;
}

static bool closed_all(const Ctx* c) { return c->cfg.n_slices && c->t >= c->cfg.n_slices; }

asse_status asse_scan_slice(void* ctx, const uint32_t* d_pairs, uint64_t n_pairs, void* stream) {
  NvtxRange nvtx_("asse_scan_slice");
  if (!ctx) return ASSE_E_PARAM;
  Ctx* c = static_cast<Ctx*>(ctx);
  if (closed_all(c)) { c->err = "all n_slices closed"; return ASSE_E_STATE; }
  if (n_pairs && (!d_pairs || ((uintptr_t)d_pairs & 7))) { c->err = "d_pairs must be 8-byte aligned device memory"; return ASSE_E_PARAM; }
  CK(cudaSetDevice(c->device));
  cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
  if (st != c->stream) {
    // a caller stream first waits for everything queued on the context stream: an
    // asse_end_slice_async's k_fold still reads and clears the touch bitmap this scan writes
    CK(cudaEventRecord(c->ev_order, c->stream));
    CK(cudaStreamWaitEvent(st, c->ev_order, 0));
  }
  asse_status s = launch_scan(c, d_pairs, n_pairs, st);
  if (s != ASSE_OK) return s;
  if (st != c->stream) {
    CK(cudaEventRecord(c->ev_join, st));
    CK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  }
  return ASSE_OK;
}

asse_status asse_scan_slice_host(void* ctx, const uint32_t* h_pairs, uint64_t n_pairs) {
  NvtxRange nvtx_("asse_scan_slice_host");
  if (!ctx) return ASSE_E_PARAM;
  Ctx* c = static_cast<Ctx*>(ctx);
  if (closed_all(c)) { c->err = "all n_slices closed"; return ASSE_E_STATE; }
  if (n_pairs == 0) return ASSE_OK;
  if (!h_pairs) return ASSE_E_PARAM;
  CK(cudaSetDevice(c->device));
  if (!c->stage[0]) {
    c->stage_pairs = 8ull << 20;  // 8 Mi pairs = 64 MiB per staging buffer
    CK(cudaMalloc(&c->stage[0], c->stage_pairs * 8));
    CK(cudaMalloc(&c->stage[1], c->stage_pairs * 8));
    CK(cudaEventRecord(c->ev_scanned[0], c->stream));
    CK(cudaEventRecord(c->ev_scanned[1], c->stream));
  }
  uint64_t off = 0;
  int b = 0;
  while (off < n_pairs) {
    uint64_t m = std::min<uint64_t>(c->stage_pairs, n_pairs - off);
    // the copy into stage[b] waits for the scan that last read it
    CK(cudaStreamWaitEvent(c->copy_stream, c->ev_scanned[b], 0));
    CK(cudaMemcpyAsync(c->stage[b], h_pairs + 2 * off, m * 8, cudaMemcpyHostToDevice, c->copy_stream));
    CK(cudaEventRecord(c->ev_copied[b], c->copy_stream));
    CK(cudaStreamWaitEvent(c->stream, c->ev_copied[b], 0));
    asse_status s = launch_scan(c, c->stage[b], m, c->stream);
    if (s != ASSE_OK) return s;
    CK(cudaEventRecord(c->ev_scanned[b], c->stream));
    off += m;
    b ^= 1;
  }
  return ASSE_OK;
}

asse_status asse_attach_peers(void* ctx, void* const* touch, void* const* merged,
                              void* const* signal, void* const* exchange, uint32_t sync_mode) {
  if (!ctx) return ASSE_E_PARAM;
  Ctx* c = static_cast<Ctx*>(ctx);
  if (c->cfg.world < 2) { c->err = "attach_peers needs world >= 2"; return ASSE_E_PEER; }
  if (sync_mode > 2) { c->err = "sync_mode is 0, 1 or 2"; return ASSE_E_PARAM; }
  if (!touch || !merged || (sync_mode == 0 && !signal) || (c->shard && !exchange)) {
    c->err = "missing peer arrays"; return ASSE_E_PEER;
  }
  for (uint32_t w = 0; w < c->cfg.world; ++w) {
    if (!touch[w] || !merged[w] || (sync_mode == 0 && !signal[w]) || (c->shard && !exchange[w])) {
      c->err = "null peer pointer"; return ASSE_E_PEER;
    }
    c->peer_touch[w] = touch[w];
    c->peer_merged[w] = merged[w];
    c->peer_signal[w] = signal ? signal[w] : nullptr;
    c->peer_xchg[w] = exchange ? exchange[w] : nullptr;
  }
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  c->touch = reinterpret_cast<uint32_t*>(touch[c->cfg.rank]);
  c->merged = reinterpret_cast<uint32_t*>(merged[c->cfg.rank]);
  c->xchg = exchange ? reinterpret_cast<uint8_t*>(exchange[c->cfg.rank]) : nullptr;
  CK(cudaMemsetAsync(c->touch, 0, c->n_atv_full * c->wpa * 4, c->stream));
  if (c->xchg) CK(cudaMemsetAsync(c->xchg, 0, 64, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  c->sync_mode = sync_mode;
  c->peers = true;
  return ASSE_OK;
}

uint64_t asse_bitmap_bytes(const void* ctx) {
  if (!ctx) return 0;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  return c->n_atv_full * c->wpa * 4;
}

uint64_t asse_merged_bytes(const void* ctx) {
  if (!ctx) return 0;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  return c->n_atv * c->wpa * 4;
}

uint64_t asse_exchange_bytes(const void* ctx) {
  if (!ctx) return 0;
  return 64 + (uint64_t)static_cast<const Ctx*>(ctx)->cfg.max_candidates * sizeof(ReportDev);
}

asse_status asse_merge(void* ctx) {
  NvtxRange nvtx_("asse_merge");
  if (!ctx) return ASSE_E_PARAM;
  Ctx* c = static_cast<Ctx*>(ctx);
  NOT_PENDING(c);
  if (!c->peers) { c->err = "asse_merge without attached peers"; return ASSE_E_PEER; }
  CK(cudaSetDevice(c->device));
  return do_merge(c);
}

static asse_status copy_reports(Ctx* c, asse_report* h_out, uint32_t cap, uint32_t* n_out, uint32_t mode) {
  const uint32_t n = (mode == 0) ? c->last_above : c->last_n;
  if (n_out) *n_out = n;
  if (!h_out || n == 0) return (h_out == nullptr && n > cap) ? ASSE_E_CAPACITY : ASSE_OK;
  if (n > cap) return ASSE_E_CAPACITY;
  if (c->h_rep_cap < n) {
    if (c->h_rep) cudaFreeHost(c->h_rep);
    c->h_rep = nullptr;
    c->h_rep_cap = std::max<uint64_t>(n, 4096);
    CK(cudaMallocHost(&c->h_rep, c->h_rep_cap * sizeof(ReportDev)));
  }
  const ReportDev* src = (mode == 0) ? c->rep_above : c->rep_sorted;
  CK(cudaMemcpyAsync(c->h_rep, src, (size_t)n * sizeof(ReportDev), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  static_assert(sizeof(ReportDev) == sizeof(asse_report), "report layout");
  memcpy(h_out, c->h_rep, (size_t)n * sizeof(ReportDev));
  return ASSE_OK;
}

// a7 + a8: restore (Alg. 4, parts CTAs per frame) with NAT and Eq. 5 fused, then the
// sort by ip; both are launched with programmatic dependent launch so their launch
// overlaps the previous kernel's tail (griddepcontrol.wait inside).
static asse_status enqueue_restore(Ctx* c) {
  cudaStream_t s = c->stream;
  RestoreParams rp = c->rp0;
  rp.sa_cnt = c->sa_cnt; rp.sa_list = c->sa_list; rp.sa_bits = c->sa_bits;
  rp.ws = c->ws; rp.ws_cap = c->ws_cap;
  rp.cand = c->cand; rp.n_cand = c->counters + 0; rp.overflow = c->counters + 1;
  rp.active = c->active; rp.aat = c->aat; rp.reports = c->rep; rp.keys = c->keys; rp.vals = c->vals;
  if (c->shard) {                   // publish this rank's reports in its exchange buffer
    rp.n_cand = reinterpret_cast<uint32_t*>(c->xchg);
    rp.reports = c->xchg + 64;
  }
  CK(launch_pdl(k_restore, dim3(c->Fl * rp.parts), dim3(512), c->restore_smem, s, rp));
  return ASSE_OK;
}
// option S: clear this rank's whole touch bitmap (every peer has merged from it) and
// gather every rank's reports
static asse_status enqueue_gather(Ctx* c) {
  cudaStream_t s = c->stream;
  CK(cudaMemsetAsync(c->touch, 0, c->n_atv_full * c->wpa * 4, s));
  GatherParams gp{};
  for (uint32_t w = 0; w < c->cfg.world; ++w) gp.xchg[w] = reinterpret_cast<const uint8_t*>(c->peer_xchg[w]);
  gp.world = c->cfg.world; gp.max_cand = c->cfg.max_candidates;
  gp.rep = c->rep; gp.keys = c->keys; gp.vals = c->vals; gp.counters = c->counters;
  k_gather_peers<<<(unsigned)c->sms, 256, 0, s>>>(gp);
  CK(cudaGetLastError());
  LAUNCHED(c);
  return ASSE_OK;
}
// Bucket sort of CSIP (k_bs_*, asse_kernels.cuh) for |CSIP| > kRankCap, |CSIP| read on the
// device; `bound` (an expected |CSIP|) only sizes the buckets (~32 ips per bucket).
static asse_status enqueue_bucket_sort(Ctx* c, const uint32_t* n_ptr, uint64_t bound, cudaStream_t s) {
  uint32_t lgB = 6;
  while (lgB < kBsMaxLgB && (1ull << lgB) * 32 < bound) ++lgB;
  if (const char* e = getenv("ASSE_BS_LGB")) lgB = std::min<uint32_t>(kBsMaxLgB, std::max(1, atoi(e)));   // tests: crowded buckets
  BucketSortParams bp{};
  bp.rep = c->rep; bp.keys = c->keys; bp.vals = c->vals; bp.n_ptr = n_ptr;
  bp.max_cand = c->cfg.max_candidates; bp.B = 1u << lgB; bp.shift = 32u - lgB;
  bp.cnt = c->bs_buf; bp.off = bp.cnt + kBsMaxB; bp.cur = bp.off + kBsMaxB;
  bp.acnt = bp.cur + kBsMaxB; bp.aoff = bp.acnt + kBsMaxB;
  bp.arank = bp.aoff + kBsMaxB; bp.pbkt = bp.arank + c->cfg.max_candidates;
  bp.tk = c->keys_alt; bp.tv = c->vals_alt;
  bp.sorted = c->rep_sorted; bp.above = c->rep_above; bp.counters = c->counters;
  const unsigned grid = (unsigned)c->sms * 4;
  CK(cudaMemsetAsync(bp.cnt, 0, (size_t)bp.B * 4, s));
  k_bs_count<<<grid, 256, 0, s>>>(bp);
  k_bs_scan<<<1, 1024, 0, s>>>(bp);
  k_bs_scatter<<<grid, 256, 0, s>>>(bp);
  k_bs_bucket<<<(bp.B + kBsWarps - 1) / kBsWarps, 32 * kBsWarps, 0, s>>>(bp);
  k_bs_scan2<<<1, 1024, 0, s>>>(bp);
  k_bs_above<<<grid, 256, 0, s>>>(bp);
  CK(cudaGetLastError());
  return ASSE_OK;
}

static asse_status enqueue_sort(Ctx* c) {
  const uint32_t* n_ptr = c->counters + (c->shard ? 6 : 0);
  CK(launch_pdl(k_sort, dim3(kSortBlocks), dim3(kSortThreads), 0, c->stream, (const ReportDev*)c->rep,
                c->counters, n_ptr, (uint32_t)c->cfg.max_candidates, c->rep_sorted, c->rep_above,
                c->sort_advances_clock ? c->d_clock : nullptr, c->two_k));
  // |CSIP| beyond the rank sort was seen: the bucket sort runs in the graph from then on
  // (its kernels return at once while |CSIP| <= kRankCap)
  if (c->sort_bound > kRankCap) return enqueue_bucket_sort(c, n_ptr, c->sort_bound, c->stream);
  return ASSE_OK;
}

static void drop_graphs(Ctx* c) {
  for (auto& row : c->graph)
    for (auto& g : row)
      if (g) { cudaGraphExecDestroy(g); g = nullptr; }
}
static asse_status enqueue_tail(Ctx* c) {
  asse_status st = enqueue_restore(c);
  if (st != ASSE_OK) return st;
  return enqueue_sort(c);
}

static FoldParams fold_params(Ctx* c, const uint32_t* src, uint32_t kp) {
  const asse_config& p = c->cfg;
  FoldParams fp{};
  fp.pool = c->pool;
  fp.touch_src = src;
  // option S: peers still read this rank's whole touch bitmap; it is cleared after the
  // second barrier (enqueue_gather), so the fold clears its (rewritten) merged input
  fp.touch_zero = c->shard ? c->merged : c->touch;
  fp.active = c->active;
  fp.aat = c->aat;
  fp.sa_cnt = c->sa_cnt;
  fp.sa_list = c->sa_list;
  fp.sa_bits = c->sa_bits;
  fp.n_super = c->counters + 3;
  fp.n_chunks = c->n_at / 512;
  fp.C0 = c->d_clock;
  fp.g = p.g; fp.k = p.k; fp.kp = kp; fp.a = c->a;
  fp.c = p.c; fp.w_theta = c->w_theta; fp.lpa_log2 = c->lpa_log2;
  return fp;
}
static unsigned fold_blocks(const Ctx* c) {
  const uint64_t tiles = (c->n_at / 512 + kFoldChunksPerTile - 1) / kFoldChunksPerTile;
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(tiles, (uint64_t)c->fold_grid));
}

// Every device operation of end_slice up to the result copies, in stream order. Used
// eagerly (world > 1 with a device barrier) or captured once into a CUDA graph per
// (timing, mode) and replayed every slice; the per-slice ACT base comes from d_clock.
static asse_status enqueue_end_slice(Ctx* c, uint32_t mode, bool timing, bool capturing) {
  cudaStream_t s = c->stream;
  // events recorded inside a captured graph must be external event-record nodes
  auto rec = [&](int i) {
    return capturing ? cudaEventRecordWithFlags(c->ev[i], s, cudaEventRecordExternal)
                     : cudaEventRecord(c->ev[i], s);
  };
  if (timing) CK(rec(0));
  // a5: merge (world > 1)
  const uint32_t* src = c->touch;
  asse_status st;
  if (c->peers) {
    if (c->sync_mode != 1) {
      if ((st = rank_barrier(c)) != ASSE_OK) return st;   // every rank's scans (and gathers) done
      if (c->shard) CK(cudaMemsetAsync(c->xchg, 0, 64, s));   // exchange count of this slice
      if ((st = do_merge(c)) != ASSE_OK) return st;
      if (!c->shard && (st = rank_barrier(c)) != ASSE_OK) return st;   // every shard merged
    }
    src = c->merged;
  }
  if (timing) CK(rec(1));
  if (c->shard && c->sync_mode == 1) {
    // option S, caller-ordered: fold + restore already ran in asse_end_slice_begin
    if (!c->begun) { c->err = "frame_shard with sync_mode 1: call asse_end_slice_begin first"; return ASSE_E_STATE; }
  } else {
    // a6: fold + weights + super + preserve(t+1)
    CK(cudaMemsetAsync(c->scratch, 0, c->scratch_bytes, s));   // AAT, SA counts/bits, counters
    const FoldParams fp = fold_params(c, src, c->kp);
    if (timing) CK(rec(2));
    if (c->cb == 1) launch_fold<1>(c->lpa_log2, c->q_log2, fold_blocks(c), s, fp);
    else launch_fold<2>(c->lpa_log2, c->q_log2, fold_blocks(c), s, fp);
    CK(cudaGetLastError());
    if (timing) CK(rec(3));
    if ((st = enqueue_restore(c)) != ASSE_OK) return st;
  }
  if (c->shard) {
    if (c->sync_mode != 1 && (st = rank_barrier(c)) != ASSE_OK) return st;   // all merged + published
    if ((st = enqueue_gather(c)) != ASSE_OK) return st;
  }
  if ((st = enqueue_sort(c)) != ASSE_OK) return st;
  if (timing) CK(rec(8));
  return ASSE_OK;
}
static constexpr int kEndSliceKernels = 3;   // fold, restore (+NAT), sort

// Copies the counters and a K-report prefix, synchronises once, runs the device-wide
// sort when |CSIP| exceeds the block sort, records statistics, advances the clock
// when closing a slice (a9), and hands the reports to the caller.
// results: counters plus a prefix of the requested report array, copied behind the slice's
// kernels; ev_collect marks their arrival. With advance the slice counts as closed here
// (a9: t+1, C0; preserveAT for t+1 was applied by k_fold, Alg. 2), so the next slice's
// scans may be issued before the results are read.
// The copies run on their own stream (d2h_stream), so the next slice's scan, queued on the
// context stream behind this slice's kernels, does not wait for them; the next end_slice
// waits for them (ev_collect) before its kernels overwrite the counters and reports.
static asse_status collect_enqueue(Ctx* c, uint32_t mode, uint32_t K, bool advance) {
  cudaStream_t s = c->stream, d = c->d2h_stream;
  CK(cudaEventRecord(c->ev_done, s));
  CK(cudaStreamWaitEvent(d, c->ev_done, 0));
  CK(cudaMemcpyAsync(c->h_counters, c->counters, 64, cudaMemcpyDeviceToHost, d));
  CK(cudaMemcpyAsync(c->h_rep, mode ? c->rep_sorted : c->rep_above, (size_t)K * sizeof(ReportDev),
                     cudaMemcpyDeviceToHost, d));
  if (c->timing && advance) CK(cudaEventRecord(c->ev[9], d));
  CK(cudaEventRecord(c->ev_collect, d));
  c->collect_pending = true;
  if (advance) {
    // merge / barrier / gather kernels of the eager multi-rank path count themselves
    c->stats.kernel_launches += kEndSliceKernels +
                                (c->sort_bound > kRankCap ? kBsKernels : 0);   // the bucket sort
    c->stats.fold_launches++;
    c->t += 1;
    c->C0 = (uint32_t)(c->t % c->two_k);
    c->stats.slices_closed++;
  }
  return ASSE_OK;
}

static asse_status collect_finish(Ctx* c, uint32_t mode, uint32_t K, asse_report* h_out, uint32_t cap,
                                  uint32_t* n_out, bool advance) {
  const asse_config& p = c->cfg;
  cudaStream_t s = c->stream;
  CK(cudaEventSynchronize(c->ev_collect));
  const uint32_t n_cand_raw = c->h_counters[c->shard ? 6 : 0];
  const bool overflow = c->h_counters[1] != 0 || n_cand_raw > p.max_candidates;
  const uint32_t n_cand = overflow ? 0 : n_cand_raw;
  bool prefetched = true;
  if (!overflow && c->h_counters[5]) {
    // |CSIP| above the rank sort and the bucket sort not yet in the graph: run it now
    const uint32_t* n_ptr = c->counters + (c->shard ? 6 : 0);
    if (asse_status e = enqueue_bucket_sort(c, n_ptr, n_cand, s)) return e;
    c->stats.kernel_launches += kBsKernels;
    CK(cudaMemcpyAsync(c->h_counters, c->counters, 64, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    prefetched = false;
    // later slices sort on the device inside the end_slice graph (buckets sized for 1.5 n)
    c->sort_bound = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(2ull * kRankCap, (uint64_t)n_cand + n_cand / 2),
                                                 p.max_candidates);
    drop_graphs(c);
  }
  if (c->sort_bound > kRankCap && n_cand > c->sort_bound) {
    // |CSIP| outgrew the bucket sort's sizing (~32 ips per bucket): resize for later slices
    c->sort_bound = (uint32_t)std::min<uint64_t>((uint64_t)n_cand + n_cand / 2, p.max_candidates);
    drop_graphs(c);
  }
  c->last_n = n_cand;
  c->last_above = n_cand ? c->h_counters[4] : 0;
  c->have_reports = true;
  c->stats.last_n_super = c->h_counters[3];
  c->stats.last_n_candidates = n_cand_raw;
  c->stats.last_n_above = c->last_above;
  if (c->timing && advance) {
    float ms;
    CK(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1])); c->stats.last_merge_ms = ms;
    CK(cudaEventElapsedTime(&ms, c->ev[2], c->ev[3])); c->stats.last_fold_ms = ms;
    c->stats.fold_ms_total += ms;
    // restore + NAT + sort run back to back under programmatic dependent launch
    CK(cudaEventElapsedTime(&ms, c->ev[3], c->ev[8])); c->stats.last_restore_ms = ms;
    c->stats.last_nat_ms = 0;
    c->stats.last_sort_ms = 0;
    CK(cudaEventElapsedTime(&ms, c->ev[0], c->ev[9])); c->stats.last_end_slice_ms = ms;
    asse_status hs = harvest_scan_timing(c);
    if (hs != ASSE_OK) return hs;
  }

  if (overflow) {
    c->last_n = c->last_above = 0;
    c->err = "CSIP exceeded max_candidates (or the restore join workspace)";
    return ASSE_E_OVERFLOW;
  }
  const uint32_t n = mode ? c->last_n : c->last_above;
  if (prefetched && n <= K) {
    if (n_out) *n_out = n;
    if (!h_out) return n > cap ? ASSE_E_CAPACITY : ASSE_OK;
    if (n > cap) return ASSE_E_CAPACITY;
    memcpy(h_out, c->h_rep, (size_t)n * sizeof(ReportDev));
    return ASSE_OK;
  }
  return copy_reports(c, h_out, cap, n_out, mode);
}

static asse_status collect(Ctx* c, uint32_t mode, uint32_t K, asse_report* h_out, uint32_t cap,
                           uint32_t* n_out, bool advance) {
  asse_status st = collect_enqueue(c, mode, K, advance);
  if (st != ASSE_OK) return st;
  return collect_finish(c, mode, K, h_out, cap, n_out, advance);
}

asse_status asse_end_slice_begin(void* ctx) {
  NvtxRange nvtx_("asse_end_slice_begin");
  if (!ctx) return ASSE_E_PARAM;
  Ctx* c = static_cast<Ctx*>(ctx);
  NOT_PENDING(c);
  if (!c->shard || !c->peers || c->sync_mode != 1) {
    c->err = "asse_end_slice_begin is for frame_shard contexts with sync_mode 1";
    return ASSE_E_STATE;
  }
  if (closed_all(c)) { c->err = "all n_slices closed"; return ASSE_E_STATE; }
  CK(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  if (c->collect_pending) CK(cudaStreamWaitEvent(s, c->ev_collect, 0));
  *c->h_clock = c->C0;
  CK(cudaMemcpyAsync(c->d_clock, c->h_clock, 4, cudaMemcpyHostToDevice, s));
  c->d_clock_known = c->C0;
  CK(cudaMemsetAsync(c->xchg, 0, 64, s));
  CK(cudaMemsetAsync(c->scratch, 0, c->scratch_bytes, s));
  const FoldParams fp = fold_params(c, c->merged, c->kp);
  if (c->cb == 1) launch_fold<1>(c->lpa_log2, c->q_log2, fold_blocks(c), s, fp);
  else launch_fold<2>(c->lpa_log2, c->q_log2, fold_blocks(c), s, fp);
  CK(cudaGetLastError());
  asse_status st = enqueue_restore(c);
  if (st != ASSE_OK) return st;
  c->begun = true;
  return ASSE_OK;
}

static asse_status end_slice_enqueue(Ctx* c, uint32_t mode, uint32_t* K_out) {
  if (mode > 1) { c->err = "mode must be 0 or 1"; return ASSE_E_PARAM; }
  if (closed_all(c)) { c->err = "all n_slices closed"; return ASSE_E_STATE; }
  if (c->cfg.world > 1 && !c->peers) { c->err = "world > 1 requires asse_attach_peers"; return ASSE_E_PEER; }
  CK(cudaSetDevice(c->device));
  const asse_config& p = c->cfg;
  cudaStream_t s = c->stream;
  const bool timing = c->timing;
  // report prefix copied with the counters: enough for the last slice's count + 25 %, so a
  // stable workload never needs a second copy (and synchronisation)
  uint64_t want = std::max<uint64_t>(1024, (uint64_t)(mode ? c->last_n : c->last_above) * 5 / 4 + 64);
  want = std::min<uint64_t>(want, p.max_candidates);
  if (want > c->h_rep_cap) {
    if (c->h_rep) CK(cudaFreeHost(c->h_rep));
    c->h_rep = nullptr;
    c->h_rep_cap = std::min<uint64_t>(std::max<uint64_t>(want * 2, 4096), p.max_candidates);
    CK(cudaMallocHost(&c->h_rep, c->h_rep_cap * sizeof(ReportDev)));
  }
  const uint32_t K = (uint32_t)std::min<uint64_t>(want, c->h_rep_cap);
  // the previous slice's result copies (d2h_stream) finish before this slice's kernels
  // rewrite the counters and report arrays
  if (c->collect_pending) CK(cudaStreamWaitEvent(s, c->ev_collect, 0));
  // the per-slice ACT base reaches the kernels through device memory, so the captured
  // graph is identical for every slice (host copies stay outside the graph)
  if (c->d_clock_known != c->C0) {           // else the previous slice's k_sort advanced it
    *c->h_clock = c->C0;
    CK(cudaMemcpyAsync(c->d_clock, c->h_clock, 4, cudaMemcpyHostToDevice, s));
  }
  c->d_clock_known = ~0u;
  c->sort_advances_clock = true;
  if ((c->peers && c->sync_mode != 1) || c->shard) {
    asse_status st = enqueue_end_slice(c, mode, timing, false);   // epochs / phases change per slice
    c->begun = false;
    c->sort_advances_clock = false;
    if (st != ASSE_OK) return st;
  } else {
    cudaGraphExec_t& ge = c->graph[timing ? 1 : 0][mode];
    if (!ge) {
      cudaGraph_t g = nullptr;
      CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      asse_status st = enqueue_end_slice(c, mode, timing, true);
      c->sort_advances_clock = false;
      cudaError_t ce = cudaStreamEndCapture(s, &g);
      if (st != ASSE_OK) { if (g) cudaGraphDestroy(g); return st; }
      CK(ce);
      CK(cudaGraphInstantiate(&ge, g, 0));
      CK(cudaGraphDestroy(g));
    }
    CK(cudaGraphLaunch(ge, s));
  }
  c->sort_advances_clock = false;
  c->d_clock_known = (c->C0 + 1u) % c->two_k;   // collect_enqueue advances C0 to the same value
  *K_out = K;
  return collect_enqueue(c, mode, K, true);
}

asse_status asse_end_slice(void* ctx, asse_report* h_out, uint32_t cap, uint32_t* n_out, uint32_t mode) {
  NvtxRange nvtx_("asse_end_slice");
  if (!ctx) return ASSE_E_PARAM;
  Ctx* c = static_cast<Ctx*>(ctx);
  if (n_out) *n_out = 0;
  NOT_PENDING(c);
  uint32_t K = 0;
  asse_status st = end_slice_enqueue(c, mode, &K);
  if (st != ASSE_OK) return st;
  return collect_finish(c, mode, K, h_out, cap, n_out, true);
}

asse_status asse_end_slice_async(void* ctx, uint32_t mode) {
  NvtxRange nvtx_("asse_end_slice_async");
  if (!ctx) return ASSE_E_PARAM;
  Ctx* c = static_cast<Ctx*>(ctx);
  NOT_PENDING(c);
  uint32_t K = 0;
  asse_status st = end_slice_enqueue(c, mode, &K);
  if (st != ASSE_OK) return st;
  c->pending = true;
  c->pend_mode = mode;
  c->pend_K = K;
  return ASSE_OK;
}

asse_status asse_end_slice_wait(void* ctx, asse_report* h_out, uint32_t cap, uint32_t* n_out) {
  NvtxRange nvtx_("asse_end_slice_wait");
  if (!ctx) return ASSE_E_PARAM;
  Ctx* c = static_cast<Ctx*>(ctx);
  if (n_out) *n_out = 0;
  if (!c->pending) { c->err = "no asynchronous end_slice pending"; return ASSE_E_STATE; }
  c->pending = false;
  CK(cudaSetDevice(c->device));
  return collect_finish(c, c->pend_mode, c->pend_K, h_out, cap, n_out, true);
}

// Window query for k' < k on the closed pool (checkAT for any
// k' <= k): weights, super ATVs, restore, NAT and Eq. 5 of the window of
// the k' slices ending at the last closed slice. The pool is not modified; preserveAT
// of the advance only erased ages >= k-1 of that slice, which no k' < k window uses.
asse_status asse_query_window(void* ctx, uint32_t k_prime, asse_report* h_out, uint32_t cap,
                              uint32_t* n_out, uint32_t mode) {
  NvtxRange nvtx_("asse_query_window");
  if (!ctx) return ASSE_E_PARAM;
  Ctx* c = static_cast<Ctx*>(ctx);
  NOT_PENDING(c);
  if (n_out) *n_out = 0;
  if (mode > 1) { c->err = "mode must be 0 or 1"; return ASSE_E_PARAM; }
  if (k_prime < 1 || k_prime >= c->cfg.k) { c->err = "query window needs 1 <= k' < k"; return ASSE_E_PARAM; }
  if (c->t == 0) { c->err = "no closed slice"; return ASSE_E_STATE; }
  if (c->shard) { c->err = "asse_query_window is not available with frame_shard"; return ASSE_E_STATE; }
  CK(cudaSetDevice(c->device));
  const asse_config& p = c->cfg;
  cudaStream_t s = c->stream;
  const uint32_t K = (uint32_t)std::min<uint64_t>(c->h_rep_cap, p.max_candidates);
  if (c->collect_pending) CK(cudaStreamWaitEvent(s, c->ev_collect, 0));
  *c->h_clock = (c->C0 + c->two_k - 1) % c->two_k;          // ACT base of the last closed slice
  CK(cudaMemcpyAsync(c->d_clock, c->h_clock, 4, cudaMemcpyHostToDevice, s));
  c->d_clock_known = *c->h_clock;                            // the next end_slice re-uploads C0
  CK(cudaMemsetAsync(c->scratch, 0, c->scratch_bytes, s));
  const FoldParams fp = fold_params(c, nullptr, k_prime);
  if (c->cb == 1) launch_fold<1, true>(c->lpa_log2, c->q_log2, fold_blocks(c), s, fp);
  else launch_fold<2, true>(c->lpa_log2, c->q_log2, fold_blocks(c), s, fp);
  CK(cudaGetLastError());
  asse_status st = enqueue_tail(c);
  if (st != ASSE_OK) return st;
  c->stats.kernel_launches += 3;
  return collect(c, mode, K, h_out, cap, n_out, false);
}

asse_status asse_fetch_reports(void* ctx, asse_report* h_out, uint32_t cap, uint32_t* n_out, uint32_t mode) {
  if (!ctx) return ASSE_E_PARAM;
  Ctx* c = static_cast<Ctx*>(ctx);
  NOT_PENDING(c);
  if (!c->have_reports) { c->err = "no closed slice"; return ASSE_E_STATE; }
  if (mode > 1) return ASSE_E_PARAM;
  CK(cudaSetDevice(c->device));
  return copy_reports(c, h_out, cap, n_out, mode);
}

// ------------------------------------------------------------ checkpoint
// File: "ASSECKPT" | u32 version (3) | u32 code_bytes | u32 k, k', r, c, u, s, g, world, rank, shard,
//       mangle, pad | f64 theta | u64 seed | u64 t | u32 C0 | u32 pad | pool codes (n_at * code_bytes,
//       canonical values). Version 3 adds mangle (the key A and the host -> ATV map depend on it).
constexpr uint32_t kCkptVersion = 3;
struct CkptHeader {
  char magic[8];
  uint32_t version, code_bytes;
  uint32_t k, kp, r, c, u, s, g;
  uint32_t world, rank, shard;
  uint32_t mangle, pad0;
  double theta;
  uint64_t seed, t;
  uint32_t C0, pad1;
};

asse_status asse_save_state(void* ctx, const char* path) {
  NvtxRange nvtx_("asse_save_state");
  if (!ctx || !path) return ASSE_E_PARAM;
  Ctx* c = static_cast<Ctx*>(ctx);
  NOT_PENDING(c);
  CK(cudaSetDevice(c->device));
  CkptHeader h{};
  memcpy(h.magic, "ASSECKPT", 8);
  h.version = kCkptVersion; h.code_bytes = c->cb;
  h.world = c->cfg.world; h.rank = c->cfg.rank; h.shard = c->shard ? 1 : 0; h.mangle = c->cfg.mangle;
  h.k = c->cfg.k; h.kp = c->kp; h.r = c->cfg.r; h.c = c->cfg.c; h.u = c->cfg.u; h.s = c->cfg.s;
  h.g = c->cfg.g; h.theta = c->cfg.theta; h.seed = c->cfg.seed; h.t = c->t; h.C0 = c->C0;
  std::vector<uint8_t> buf(c->n_at * c->cb);
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaMemcpy(buf.data(), c->pool, buf.size(), cudaMemcpyDeviceToHost));
  FILE* f = fopen(path, "wb");
  if (!f) { c->err = std::string("cannot open ") + path; return ASSE_E_PARAM; }
  bool ok = fwrite(&h, sizeof(h), 1, f) == 1 && fwrite(buf.data(), 1, buf.size(), f) == buf.size();
  ok = (fclose(f) == 0) && ok;
  if (!ok) { c->err = std::string("short write to ") + path; return ASSE_E_PARAM; }
  return ASSE_OK;
}

asse_status asse_load_state(void* ctx, const char* path) {
  NvtxRange nvtx_("asse_load_state");
  if (!ctx || !path) return ASSE_E_PARAM;
  Ctx* c = static_cast<Ctx*>(ctx);
  NOT_PENDING(c);
  CK(cudaSetDevice(c->device));
  FILE* f = fopen(path, "rb");
  if (!f) { c->err = std::string("cannot open ") + path; return ASSE_E_PARAM; }
  CkptHeader h{};
  std::vector<uint8_t> buf(c->n_at * c->cb);
  bool ok = fread(&h, sizeof(h), 1, f) == 1;
  if (ok && (memcmp(h.magic, "ASSECKPT", 8) != 0 || h.version != kCkptVersion)) {
    fclose(f); c->err = "not an ASSE checkpoint (version 3)"; return ASSE_E_PARAM;
  }
  if (ok && h.mangle != c->cfg.mangle) { fclose(f); c->err = "checkpoint mangling (mangle) differs"; return ASSE_E_PARAM; }
  if (ok && (h.C0 != (uint32_t)(h.t % c->two_k) || (c->cfg.n_slices && h.t > c->cfg.n_slices))) {
    fclose(f); c->err = "checkpoint clock inconsistent: C0 != t mod 2k, or t beyond n_slices"; return ASSE_E_PARAM;
  }
  if (ok && h.shard != (c->shard ? 1u : 0u)) { fclose(f); c->err = "checkpoint frame sharding differs"; return ASSE_E_PARAM; }
  if (ok && h.shard && (h.world != c->cfg.world || h.rank != c->cfg.rank)) {
    fclose(f); c->err = "frame-sharded checkpoint of another rank/world"; return ASSE_E_PARAM;
  }
  if (ok && (h.code_bytes != c->cb || h.k != c->cfg.k || h.kp != c->kp || h.r != c->cfg.r || h.c != c->cfg.c ||
             h.u != c->cfg.u || h.s != c->cfg.s || h.g != c->cfg.g || h.theta != c->cfg.theta ||
             h.seed != c->cfg.seed)) {
    fclose(f);
    c->err = "checkpoint parameters differ from the context (k, k', r, c, u, s, g, theta, seed)";
    return ASSE_E_PARAM;
  }
  ok = ok && fread(buf.data(), 1, buf.size(), f) == buf.size();
  fclose(f);
  if (!ok) { c->err = std::string("short read from ") + path; return ASSE_E_PARAM; }
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaMemcpy(c->pool, buf.data(), buf.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(c->touch, 0, c->n_atv_full * c->wpa * 4));
  c->t = h.t;
  c->C0 = h.C0;
  c->have_reports = false;
  return ASSE_OK;
}

uint64_t asse_pool_size(const void* ctx) {
  return ctx ? static_cast<const Ctx*>(ctx)->n_at : 0;
}

asse_status asse_export_pool(void* ctx, uint16_t* h_out, uint64_t n) {
  NvtxRange nvtx_("asse_export_pool");
  if (!ctx) return ASSE_E_PARAM;
  Ctx* c = static_cast<Ctx*>(ctx);
  NOT_PENDING(c);
  if (!h_out || n != c->n_at) { c->err = "export_pool: n must equal asse_pool_size()"; return ASSE_E_PARAM; }
  CK(cudaSetDevice(c->device));
  if (c->cb == 2) {
    CK(cudaMemcpyAsync(h_out, c->pool, n * 2, cudaMemcpyDeviceToHost, c->stream));
  } else {
    if (!c->export_buf) CK(cudaMalloc(&c->export_buf, n * 2));
    uint64_t blocks = std::min<uint64_t>((n + 255) / 256, (uint64_t)c->sms * 16);
    k_export_u8<<<(unsigned)blocks, 256, 0, c->stream>>>((const uint8_t*)c->pool, c->export_buf, n);
    CK(cudaGetLastError());
    LAUNCHED(c);
    CK(cudaMemcpyAsync(h_out, c->export_buf, n * 2, cudaMemcpyDeviceToHost, c->stream));
  }
  CK(cudaStreamSynchronize(c->stream));
  return ASSE_OK;
}

asse_status asse_get_clock(const void* ctx, uint64_t* t, uint32_t* C0) {
  if (!ctx) return ASSE_E_PARAM;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  if (t) *t = c->t;
  if (C0) *C0 = c->C0;
  return ASSE_OK;
}

asse_status asse_get_keys(const void* ctx, uint64_t* A, uint64_t* A_inv, uint64_t* K_bh) {
  if (!ctx) return ASSE_E_PARAM;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  if (A) *A = c->A;
  if (A_inv) *A_inv = c->A_inv;
  if (K_bh) *K_bh = c->K_bh;
  return ASSE_OK;
}

asse_status asse_get_stats(const void* ctx, asse_stats* out) {
  if (!ctx || !out) return ASSE_E_PARAM;
  *out = static_cast<const Ctx*>(ctx)->stats;
  return ASSE_OK;
}

void* asse_get_stream(const void* ctx) {
  return ctx ? (void*)static_cast<const Ctx*>(ctx)->stream : nullptr;
}

asse_status asse_set_host_barrier(void* ctx, asse_host_barrier_fn fn, void* arg) {
  if (!ctx) return ASSE_E_PARAM;
  Ctx* c = static_cast<Ctx*>(ctx);
  c->host_barrier = fn;
  c->host_barrier_arg = arg;
  return ASSE_OK;
}

// ------------------------------------------------------------ CUDA IPC helpers
#ifdef ASSE_RESTORE_PROF
// tools only (ASSE_RESTORE_PROF build): copy the per-CTA restore timeline marks
extern "C" int asse_debug_restore_prof(unsigned long long* out, unsigned n) {
  return (int)cudaMemcpyFromSymbol(out, g_restore_prof, (size_t)n * 8 * 8);
}
#endif
static_assert(sizeof(cudaIpcMemHandle_t) == ASSE_IPC_HANDLE_BYTES, "IPC handle size");

asse_status asse_ipc_alloc(int32_t device, uint64_t bytes, void** d_ptr, uint8_t* handle) {
  if (!d_ptr || !handle || bytes == 0) return ASSE_E_PARAM;
  *d_ptr = nullptr;
  if (cudaSetDevice(device) != cudaSuccess) return ASSE_E_CUDA;
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) return ASSE_E_CUDA;
  cudaIpcMemHandle_t h;
  if (cudaMemset(p, 0, bytes) != cudaSuccess || cudaIpcGetMemHandle(&h, p) != cudaSuccess) {
    cudaFree(p);
    return ASSE_E_CUDA;
  }
  memcpy(handle, &h, sizeof(h));
  *d_ptr = p;
  return ASSE_OK;
}

asse_status asse_ipc_open(const uint8_t* handle, int32_t device, void** d_ptr) {
  if (!d_ptr || !handle) return ASSE_E_PARAM;
  *d_ptr = nullptr;
  if (cudaSetDevice(device) != cudaSuccess) return ASSE_E_CUDA;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  if (cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
    cudaGetLastError();
    return ASSE_E_PEER;
  }
  return ASSE_OK;
}

asse_status asse_ipc_free(void* d_ptr, int32_t opened) {
  if (!d_ptr) return ASSE_OK;
  cudaError_t e = opened ? cudaIpcCloseMemHandle(d_ptr) : cudaFree(d_ptr);
  return e == cudaSuccess ? ASSE_OK : ASSE_E_CUDA;
}

// Self-test of the device barrier (k_barrier's protocol) as ONE cooperative kernel whose
// blocks play the ranks: never as separate launches that wait on each other.
asse_status asse_selftest_barrier(int32_t device, uint32_t world, uint32_t epochs, uint64_t* errors) {
  if (!errors || world < 2 || world > (uint32_t)kMaxWorld || epochs == 0) return ASSE_E_PARAM;
  *errors = ~0ull;
  if (cudaSetDevice(device) != cudaSuccess) return ASSE_E_CUDA;
  uint32_t* mem = nullptr;
  const size_t pad_words = 64, words = (size_t)world * pad_words + (size_t)world * 32 + 2;
  if (cudaMalloc(&mem, words * 4) != cudaSuccess) return ASSE_E_CUDA;
  asse_status st = ASSE_OK;
  do {
    if (cudaMemset(mem, 0, words * 4) != cudaSuccess) { st = ASSE_E_CUDA; break; }
    BarrierTestParams tp{};
    for (uint32_t w = 0; w < world; ++w) tp.bp.pads[w] = mem + w * pad_words;
    tp.bp.world = world;
    tp.data = mem + world * pad_words;
    tp.errors = reinterpret_cast<unsigned long long*>(mem + world * pad_words + world * 32);
    tp.epochs = epochs;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(world);
    cfg.blockDim = dim3(32);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, k_barrier_selftest, tp) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess) { cudaGetLastError(); st = ASSE_E_CUDA; break; }
    unsigned long long e = 0;
    if (cudaMemcpy(&e, tp.errors, 8, cudaMemcpyDeviceToHost) != cudaSuccess) { st = ASSE_E_CUDA; break; }
    *errors = e;
  } while (0);
  cudaFree(mem);
  return st;
}

}  // extern "C"
