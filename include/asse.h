/*
 * asse.h — C-ABI of libasse, the B200-native (sm_100a) hot path of ASSE:
 * "Distributed super point cardinality estimation under sliding time window for
 * high speed network" (arXiv 1807.01527). Citations: P:n = line n of the paper's
 * PAPER.md; A<n> = reading n of DESIGN.md §2 (= SURVEY.md §8(c)).
 *
 * Conventions
 *  - Every function returns asse_status (0 = OK, < 0 = error); no C++ exception
 *    crosses the ABI. asse_last_error(ctx) returns a message for the last error.
 *  - A context is bound to one CUDA device and one process; it is NOT thread-safe.
 *  - The library owns every device buffer it allocates. Caller-owned memory is
 *    marked "caller-owned" below.
 *  - "Slice t" is the time slice being filled; asse_end_slice closes it.
 *
 * Device layout: AT pool codes [y][z][x][i] (u8 when 2k <= 126,
 * else u16, A2); per-slice touch bitmap and active bitmap, g bits per ATV, in
 * the same [y][z][x] order.
 */
#ifndef ASSE_H
#define ASSE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ASSE_OK = 0,
  ASSE_E_PARAM = -1,     /* invalid configuration or argument */
  ASSE_E_STATE = -2,     /* call not allowed in the current state */
  ASSE_E_CAPACITY = -3,  /* caller buffer too small; *n_out holds the needed count */
  ASSE_E_OVERFLOW = -4,  /* CSIP (or the restore join workspace) exceeded max_candidates */
  ASSE_E_CUDA = -5,      /* a CUDA runtime error (message in asse_last_error) */
  ASSE_E_PEER = -6       /* multi-GPU peers missing or inconsistent */
} asse_status;

/* Configuration (P:452 parameters; geometry reading A12). */
typedef struct {
  uint32_t k;              /* window length in slices, k >= 1 */
  uint32_t n_slices;       /* slices the run may close; 0 = unbounded */
  uint32_t r, c, u, s, g;  /* rows, column bits, frame bits, stride, ATs per ATV */
  double theta;            /* super-point threshold, >= (A22) */
  uint64_t seed;           /* master seed -> mangling key A (odd) and BH key (A14) */
  uint32_t k_prime;        /* estimate window k' <= k (Alg. 1); 0 => k (A5) */
  uint32_t max_candidates; /* CSIP capacity; also sizes the restore join workspace */
  int32_t device;          /* CUDA device ordinal */
  uint32_t world, rank;    /* multi-GPU: packets sharded across `world` ranks */
  uint32_t frame_shard;    /* 0: every rank keeps the whole pool (replicated, option R);
                              1: rank d keeps frames [d*F/world, (d+1)*F/world) (option S,
                              SURVEY §8(e)); world must divide F = 2^u */
  uint32_t mangle;         /* 0: f(aip) = A*aip mod 2^32, A odd (A8);
                              1: f(aip) = A*aip mod p, p = 2^32+15 prime, cycle-walked into
                              32 bits (P:305 literal) */
} asse_config;

/* One CSIP member (Alg. 4 output) with its Alg. 5 NAT and Eq. 5 estimate. */
typedef struct {
  uint32_t ip;             /* restored super-point candidate (f^{-1} applied) */
  uint32_t nat;            /* NAT(ip): ATs active in all r ATVs (Alg. 5) */
  double estimate;         /* Eq. 5 (A19); +inf when nat == g (A20) */
  uint32_t flags;          /* ASSE_FLAG_* */
  uint32_t pad;
} asse_report;
#define ASSE_FLAG_SATURATED 1u   /* nat == g */
#define ASSE_FLAG_ABOVE_THETA 2u /* estimate >= theta */

/* Per-context statistics (device times from CUDA events on the launching stream). */
typedef struct {
  uint64_t slices_closed;
  uint64_t packets_scanned;      /* cumulative */
  uint64_t kernel_launches;      /* cumulative count of this library's kernel launches */
  uint64_t scan_launches;        /* cumulative k_scan launches */
  double scan_ms_total;          /* cumulative k_scan device time (timing enabled only) */
  double fold_ms_total;          /* cumulative k_fold device time (timing enabled only) */
  uint64_t fold_launches;
  double last_merge_ms, last_fold_ms;
  double last_restore_ms;        /* restore + NAT/Eq. 5 + sort (launched back to back) */
  double last_nat_ms, last_sort_ms;  /* 0: fused into last_restore_ms */
  double last_end_slice_ms;      /* device time of the whole last end_slice */
  uint32_t last_n_super;         /* super ATVs in the last slice, all rows/frames */
  uint32_t last_n_candidates;    /* |CSIP| of the last slice */
  uint32_t last_n_above;         /* candidates with estimate >= theta */
  uint32_t w_theta;              /* integer super-ATV weight threshold (A15) */
  uint32_t code_bytes;           /* device AT code width: 1 or 2 (A2) */
  uint32_t scan_bin_launches;    /* cumulative launches of the binned scan (k_scan_bin) */
  uint32_t scan_rows_red;        /* k_scan_bin: rows whose SetATs take the direct RED route */
  uint32_t scan_bin_ok;          /* 1 if k_scan_bin is available for this geometry/device */
  uint32_t scan_own_launches;    /* cumulative launches of the packet-owned scan (k_scan_own) */
  uint32_t scan_own_ok;          /* 1 if k_scan_own is available for this geometry/device */
  uint32_t host_barriers;        /* cumulative host barriers (sync_mode 2) */
  uint32_t pad0;
} asse_stats;

/* Validate a configuration (completeness/redundancy P:315-324, A10). The device path
 * additionally needs g a power of two in [128, 4096], c + u <= 24, 2 <= r <= 8,
 * k <= 16383 and world <= 16 (frame_shard: world divides 2^u).
 * why: caller-owned buffer of n bytes for a message (may be NULL). */
asse_status asse_validate(const asse_config* cfg, char* why, size_t n);

/* Create a context: derive keys (A14), W_theta (A15), allocate the pool with every
 * AT = 2k (InitAT), C0 = 0, t = 0 (A3). *out receives the context. */
asse_status asse_init(const asse_config* cfg, void** out);

/* Destroy a context and free its device memory. NULL is ignored. */
void asse_destroy(void* ctx);

/* Message describing the last error on ctx (static string if ctx is NULL). */
const char* asse_last_error(const void* ctx);

/* Enable/disable per-kernel CUDA-event timing (asse_stats.*_ms). Default off. */
asse_status asse_set_timing(void* ctx, int enable);

/* Scan kernel selection: 0 = automatic (default: the packet-owned scan k_scan_own when the
 * geometry admits it — r = 4, g/32 a power of two, an owner slice of r x 2^c ATVs x g/32/NGRP
 * words fits one SM's shared memory — and a call brings at least 8 rounds of packets per SM;
 * else the binned scan k_scan_bin under the same size rule when its part of the touch bitmap
 * fits the SMs' shared memory; else k_scan), 1 = always k_scan (one RED.OR per SetAT into the
 * L2-resident bitmap), 2 = always k_scan_bin, 3 = always k_scan_own (ASSE_E_PARAM if the
 * chosen kernel is unavailable). All produce the identical touch bitmap (SetAT is
 * idempotent), so pools and reports do not depend on the choice. */
asse_status asse_set_scan_variant(void* ctx, int variant);

/* Alg. 3 "Scan IP pair" for n_pairs packets of the current slice.
 * d_pairs: caller-owned DEVICE buffer of 2*n_pairs uint32 [aip0,bip0,aip1,...]
 *          (A33), 8-byte aligned; it must stay valid until the scan has run
 *          (stream-ordered on `stream`; asse_end_slice synchronizes).
 * stream:  cudaStream_t to launch on (NULL = the context's stream). A caller stream is
 *          first made to wait for the context's stream (a pending asse_end_slice_async
 *          still folds and clears the touch bitmap), then the context's stream is made
 *          to wait on it, so end_slice sees every scan (A34). Scans of one context are
 *          serialised whatever streams they are issued on.
 * Asynchronous; may be called any number of times per slice; n_pairs = 0 is legal. */
asse_status asse_scan_slice(void* ctx, const uint32_t* d_pairs, uint64_t n_pairs, void* stream);

/* Same as asse_scan_slice for a caller-owned HOST buffer (pinned for full speed):
 * the library copies it in chunks through two device staging buffers on a copy
 * stream, overlapping each chunk's H2D copy with the previous chunk's scan
 * (the paper's double buffering). Returns after the last copy is issued;
 * the host buffer must stay valid until asse_end_slice returns. */
asse_status asse_scan_slice_host(void* ctx, const uint32_t* h_pairs, uint64_t n_pairs);

/* Close slice t: (world > 1: merge the touch bitmaps of all ranks, A26), fold the
 * slice's SetATs into the pool, weights |ATV|^{k'} and AAT, super
 * ATVs, restore CSIP (Alg. 4), NAT + Eq. 5 (Alg. 5), sort by ip (A24), then
 * advance to t+1 with preserveAT on the blocks whose ACT becomes 0 or k (Alg. 2).
 * mode 0: reports with estimate >= theta (A21); mode 1: every CSIP member.
 * h_out: caller-owned host array of cap reports (may be NULL with cap 0 to query).
 * *n_out: number of reports produced. If cap < *n_out returns ASSE_E_CAPACITY
 * (the slice is still closed; asse_fetch_reports re-reads the reports).
 * ASSE_E_OVERFLOW: CSIP exceeded max_candidates; the slice is still closed and the
 * pool advanced, *n_out = 0. ASSE_E_STATE after n_slices closed slices. Synchronous. */
asse_status asse_end_slice(void* ctx, asse_report* h_out, uint32_t cap, uint32_t* n_out,
                           uint32_t mode);

/* Asynchronous asse_end_slice, for pipelining slices: enqueues everything asse_end_slice
 * does (merge, fold, restore, NAT/Eq. 5, sort, the copy of the counters and of a report
 * prefix to pinned host memory) on the context's stream and returns at once. The slice
 * counts as closed on return (t+1, C0 advanced), so the next slice's asse_scan_slice may
 * be issued before its results are read; the device runs the scans after this slice's
 * kernels (stream order). At most one slice may be pending: asse_end_slice_wait must be
 * called before the next asse_end_slice(_async), query, fetch, export, save/load or merge
 * (those return ASSE_E_STATE meanwhile). Errors of the slice itself (ASSE_E_OVERFLOW,
 * ASSE_E_CAPACITY) are reported by asse_end_slice_wait. */
asse_status asse_end_slice_async(void* ctx, uint32_t mode);

/* Wait for the pending asynchronous end_slice and return its reports with the same
 * conventions as asse_end_slice (h_out caller-owned host array of cap reports, *n_out
 * produced; mode was given to asse_end_slice_async). ASSE_E_STATE if none is pending. */
asse_status asse_end_slice_wait(void* ctx, asse_report* h_out, uint32_t cap, uint32_t* n_out);

/* Window query (checkAT for any k' <= k): super
 * points and Eq. 5 estimates over the k_prime slices ending at the last closed slice,
 * evaluated on the current pool without modifying it. 1 <= k_prime < k (the advance's
 * preserveAT has erased ages >= k-1 of that slice, which only the k' = k window uses;
 * k' = k is what asse_end_slice returns with k_prime = 0). Needs >= 1 closed slice;
 * pending scans of the next slice are ignored. Same output conventions as
 * asse_end_slice; afterwards asse_fetch_reports returns this query's reports. */
asse_status asse_query_window(void* ctx, uint32_t k_prime, asse_report* h_out, uint32_t cap,
                              uint32_t* n_out, uint32_t mode);

/* Re-read the reports of the last closed slice (same mode semantics). */
asse_status asse_fetch_reports(void* ctx, asse_report* h_out, uint32_t cap, uint32_t* n_out,
                               uint32_t mode);

/* Export the AT pool in the canonical layout [y][z][x][i], one uint16 per AT
 * (values in [0, 2k], 2k = inactive). h_out: caller-owned host array of n entries,
 * n must equal asse_pool_size() (r * 2^u * 2^c * g; in option S only this rank's frames,
 * [y][z - z_first][x][i]). Reflects the state after the last end_slice
 * (post-advance, A32) plus any scans issued since (not yet folded: excluded). */
asse_status asse_export_pool(void* ctx, uint16_t* h_out, uint64_t n);

/* Checkpoint: write the pool codes, slice index t and ACT
 * base C0 with the parameters (k, k', r, c, u, s, g, theta, seed, mangle, frame sharding)
 * and a magic/version (3) header to `path`. Take it after asse_end_slice (touches of a slice still being
 * scanned are not saved). ASSE_E_PARAM on I/O errors. */
asse_status asse_save_state(void* ctx, const char* path);

/* Restore a checkpoint into a context created with the same parameters (rejects any
 * parameter mismatch, another version, or a clock with C0 != t mod 2k, with ASSE_E_PARAM);
 * pending touches of the context are discarded. */
asse_status asse_load_state(void* ctx, const char* path);

/* Number of ATs in this context's pool (r * 2^u * 2^c * g, or its frames' share in option S). */
uint64_t asse_pool_size(const void* ctx);

/* Current slice index t and ACT base C0. */
asse_status asse_get_clock(const void* ctx, uint64_t* t, uint32_t* C0);

/* Keys derived from the seed (A14): A, A^{-1} (mod 2^32, or mod p with mangle = 1), K_bh. */
asse_status asse_get_keys(const void* ctx, uint64_t* A, uint64_t* A_inv, uint64_t* K_bh);

/* Statistics; out: caller-owned asse_stats. */
asse_status asse_get_stats(const void* ctx, asse_stats* out);

/* The context's CUDA stream (cudaStream_t). */
void* asse_get_stream(const void* ctx);

/* Multi-GPU. world = cfg.world ranks, this rank = cfg.rank.
 * touch[w]:  device pointers (peer-mapped, e.g. torch symmetric memory) of every
 *            rank's per-slice touch bitmap, each asse_bitmap_bytes() long; touch[rank]
 *            replaces this context's own touch bitmap.
 * merged[w]: every rank's merged bitmap, asse_merged_bytes() long (the whole geometry
 *            in option R, the rank's own frames in option S).
 * exchange[w]: option S only (else NULL): every rank's report exchange buffer,
 *            asse_exchange_bytes() long; each rank publishes its frames' reports there
 *            and gathers every peer's.
 * signal[w]: every rank's signal pad (>= 256 bytes, zero-initialised) used by the
 *            stream-ordered cross-GPU barrier when sync_mode == 0.
 * sync_mode: 0 = device barrier over the signal pads (one process per GPU);
 *            1 = caller-ordered (all ranks' scans complete before any merge, all
 *                merges complete before any end_slice; used by single-GPU tests);
 *            2 = host barrier: at each cross-rank point end_slice synchronises the
 *                context's stream and calls the callback set by asse_set_host_barrier
 *                (e.g. a torch.distributed barrier); no kernel waits on another rank's
 *                kernel, so ranks may share a GPU. signal may be NULL.
 * Buffers are caller-owned and must outlive the context. */
asse_status asse_attach_peers(void* ctx, void* const* touch, void* const* merged,
                              void* const* signal, void* const* exchange, uint32_t sync_mode);

/* sync_mode 2: the host barrier across all ranks. fn(arg) must return 0 after every rank
 * has called it for the same barrier instance (nonzero: end_slice fails with ASSE_E_PEER).
 * end_slice calls it 2 times per slice (option R: before the merge, after the merge;
 * option S: before the merge, before the report gather). */
typedef int (*asse_host_barrier_fn)(void* arg);
asse_status asse_set_host_barrier(void* ctx, asse_host_barrier_fn fn, void* arg);

/* CUDA IPC peer buffers (one process per rank on one node; NVLink peer access is enabled
 * lazily on open). asse_ipc_alloc: zeroed device buffer of `bytes` on `device` (library-
 * owned until asse_ipc_free(ptr, 0)) and its 64-byte handle (caller-owned `handle`);
 * asse_ipc_open: map another process's buffer, released with asse_ipc_free(ptr, 1).
 * A process cannot open its own handle (ASSE_E_PEER). */
#define ASSE_IPC_HANDLE_BYTES 64
asse_status asse_ipc_alloc(int32_t device, uint64_t bytes, void** d_ptr, uint8_t* handle);
asse_status asse_ipc_open(const uint8_t* handle, int32_t device, void** d_ptr);
asse_status asse_ipc_free(void* d_ptr, int32_t opened);

/* Self-test of the cross-rank device barrier used by sync_mode 0 (k_barrier): `world`
 * ranks are played by the blocks of ONE cooperative kernel on `device` (co-resident by
 * construction), each crossing 2 * epochs barriers and checking after each that it sees
 * every rank's data of that epoch. *errors = number of stale reads (0 = pass). */
asse_status asse_selftest_barrier(int32_t device, uint32_t world, uint32_t epochs, uint64_t* errors);

/* Bytes of one touch bitmap (whole geometry): r * 2^u * 2^c * g / 8. */
uint64_t asse_bitmap_bytes(const void* ctx);

/* Bytes of this rank's merged bitmap (its frames only in option S). */
uint64_t asse_merged_bytes(const void* ctx);

/* Bytes of one report exchange buffer (option S): 64 + max_candidates * sizeof(asse_report). */
uint64_t asse_exchange_bytes(const void* ctx);

/* Option S with sync_mode 1 (caller-ordered phases on one GPU): after asse_merge on every
 * rank, fold + restore + NAT of this rank's frames, publishing its reports in its exchange
 * buffer; then asse_end_slice on every rank gathers all ranks' reports. */
asse_status asse_end_slice_begin(void* ctx);

/* Multi-GPU phase 1 of end_slice (called by asse_end_slice itself when sync_mode
 * == 0): OR this rank's 1/world shard of every rank's touch bitmap and store the
 * result into every rank's merged bitmap (reduce-scatter + all-gather in one
 * peer-memory kernel). With sync_mode 1 the caller runs it for every rank, then
 * synchronizes, then calls asse_end_slice for every rank. */
asse_status asse_merge(void* ctx);

#ifdef __cplusplus
}
#endif
#endif /* ASSE_H */
