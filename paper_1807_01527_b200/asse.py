"""ctypes binding of libasse (include/asse.h) — argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module never
computes anything of the method and has no CPU fallback: if libasse.so is
missing or a CUDA call fails it raises.
"""
import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libasse.so")

REPORT_DTYPE = np.dtype([("ip", "<u4"), ("nat", "<u4"), ("estimate", "<f8"),
                         ("flags", "<u4"), ("pad", "<u4")])
FLAG_SATURATED, FLAG_ABOVE_THETA = 1, 2

OK, E_PARAM, E_STATE, E_CAPACITY, E_OVERFLOW, E_CUDA, E_PEER = 0, -1, -2, -3, -4, -5, -6
_NAMES = {E_PARAM: "ASSE_E_PARAM", E_STATE: "ASSE_E_STATE", E_CAPACITY: "ASSE_E_CAPACITY",
          E_OVERFLOW: "ASSE_E_OVERFLOW", E_CUDA: "ASSE_E_CUDA", E_PEER: "ASSE_E_PEER"}

# every symbol include/asse.h declares
SYMBOLS = ["asse_validate", "asse_init", "asse_destroy", "asse_last_error", "asse_set_timing", "asse_set_scan_variant",
           "asse_scan_slice", "asse_scan_slice_host", "asse_end_slice", "asse_fetch_reports",
           "asse_export_pool", "asse_pool_size", "asse_get_clock", "asse_get_keys",
           "asse_get_stats", "asse_get_stream", "asse_attach_peers", "asse_bitmap_bytes",
           "asse_merge", "asse_query_window", "asse_save_state", "asse_load_state",
           "asse_merged_bytes", "asse_exchange_bytes", "asse_end_slice_begin", "asse_end_slice_async",
           "asse_end_slice_wait", "asse_set_host_barrier", "asse_ipc_alloc", "asse_ipc_open",
           "asse_ipc_free", "asse_selftest_barrier"]


class AsseError(RuntimeError):
    def __init__(self, status, msg=""):
        super().__init__("%s: %s" % (_NAMES.get(status, status), msg))
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [("k", ctypes.c_uint32), ("n_slices", ctypes.c_uint32),
                ("r", ctypes.c_uint32), ("c", ctypes.c_uint32), ("u", ctypes.c_uint32),
                ("s", ctypes.c_uint32), ("g", ctypes.c_uint32), ("theta", ctypes.c_double),
                ("seed", ctypes.c_uint64), ("k_prime", ctypes.c_uint32),
                ("max_candidates", ctypes.c_uint32), ("device", ctypes.c_int32),
                ("world", ctypes.c_uint32), ("rank", ctypes.c_uint32),
                ("frame_shard", ctypes.c_uint32), ("mangle", ctypes.c_uint32)]


class Stats(ctypes.Structure):
    _fields_ = [("slices_closed", ctypes.c_uint64), ("packets_scanned", ctypes.c_uint64),
                ("kernel_launches", ctypes.c_uint64), ("scan_launches", ctypes.c_uint64),
                ("scan_ms_total", ctypes.c_double), ("fold_ms_total", ctypes.c_double),
                ("fold_launches", ctypes.c_uint64),
                ("last_merge_ms", ctypes.c_double), ("last_fold_ms", ctypes.c_double),
                ("last_restore_ms", ctypes.c_double), ("last_nat_ms", ctypes.c_double),
                ("last_sort_ms", ctypes.c_double), ("last_end_slice_ms", ctypes.c_double),
                ("last_n_super", ctypes.c_uint32), ("last_n_candidates", ctypes.c_uint32),
                ("last_n_above", ctypes.c_uint32), ("w_theta", ctypes.c_uint32),
                ("code_bytes", ctypes.c_uint32), ("scan_bin_launches", ctypes.c_uint32),
                ("scan_rows_red", ctypes.c_uint32), ("scan_bin_ok", ctypes.c_uint32),
                ("scan_own_launches", ctypes.c_uint32), ("scan_own_ok", ctypes.c_uint32),
                ("host_barriers", ctypes.c_uint32), ("pad", ctypes.c_uint32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_ if f != "pad"}


_lib = None
HOST_BARRIER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p)
IPC_HANDLE_BYTES = 64


def load_library(path=None):
    """Load libasse.so (raises if it is missing — there is no fallback). ASSE_LIB may name
    another build of the same library (tools/sweep.py: kernel variants built out of tree,
    never copied over the product .so)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("ASSE_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise ImportError("libasse.so not built (%s); run __graft_entry__.build()" % path)
    L = ctypes.CDLL(path)
    vp, u32, u64, i32 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
    C = ctypes.POINTER(Config)
    sigs = {
        "asse_validate": (i32, [C, ctypes.c_char_p, ctypes.c_size_t]),
        "asse_init": (i32, [C, ctypes.POINTER(vp)]),
        "asse_destroy": (None, [vp]),
        "asse_last_error": (ctypes.c_char_p, [vp]),
        "asse_set_timing": (i32, [vp, i32]),
        "asse_set_scan_variant": (i32, [vp, i32]),
        "asse_scan_slice": (i32, [vp, vp, u64, vp]),
        "asse_scan_slice_host": (i32, [vp, vp, u64]),
        "asse_end_slice": (i32, [vp, vp, u32, ctypes.POINTER(u32), u32]),
        "asse_end_slice_async": (i32, [vp, u32]),
        "asse_end_slice_wait": (i32, [vp, vp, u32, ctypes.POINTER(u32)]),
        "asse_fetch_reports": (i32, [vp, vp, u32, ctypes.POINTER(u32), u32]),
        "asse_export_pool": (i32, [vp, vp, u64]),
        "asse_pool_size": (u64, [vp]),
        "asse_get_clock": (i32, [vp, ctypes.POINTER(u64), ctypes.POINTER(u32)]),
        "asse_get_keys": (i32, [vp, ctypes.POINTER(u64), ctypes.POINTER(u64), ctypes.POINTER(u64)]),
        "asse_get_stats": (i32, [vp, ctypes.POINTER(Stats)]),
        "asse_get_stream": (vp, [vp]),
        "asse_attach_peers": (i32, [vp, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp),
                                    ctypes.POINTER(vp), u32]),
        "asse_merged_bytes": (u64, [vp]),
        "asse_exchange_bytes": (u64, [vp]),
        "asse_end_slice_begin": (i32, [vp]),
        "asse_bitmap_bytes": (u64, [vp]),
        "asse_merge": (i32, [vp]),
        "asse_query_window": (i32, [vp, u32, vp, u32, ctypes.POINTER(u32), u32]),
        "asse_save_state": (i32, [vp, ctypes.c_char_p]),
        "asse_load_state": (i32, [vp, ctypes.c_char_p]),
        "asse_set_host_barrier": (i32, [vp, HOST_BARRIER_FN, vp]),
        "asse_ipc_alloc": (i32, [i32, u64, ctypes.POINTER(vp), ctypes.c_char_p]),
        "asse_ipc_open": (i32, [ctypes.c_char_p, i32, ctypes.POINTER(vp)]),
        "asse_ipc_free": (i32, [vp, i32]),
        "asse_selftest_barrier": (i32, [i32, u32, u32, ctypes.POINTER(u64)]),
    }
    for name, (rt, at) in sigs.items():
        f = getattr(L, name)
        f.restype, f.argtypes = rt, at
    _lib = L
    return L


def make_config(k, r, c, u, s, g, theta, seed, k_prime=0, n_slices=0, max_candidates=1 << 20,
                device=0, world=1, rank=0, frame_shard=0, mangle=0, **_):
    return Config(k, n_slices, r, c, u, s, g, float(theta), seed, k_prime, max_candidates,
                  device, world, rank, frame_shard, mangle)


def validate(**kw):
    why = ctypes.create_string_buffer(256)
    cfg = make_config(**kw)
    return load_library().asse_validate(ctypes.byref(cfg), why, 256), why.value.decode()


class Asse:
    """One ASSE context on one GPU. Keyword geometry as in gen.PRESETS."""

    def __init__(self, **kw):
        self._L = load_library()
        self.cfg = make_config(**kw)
        self.kw = dict(kw)
        h = ctypes.c_void_p()
        st = self._L.asse_init(ctypes.byref(self.cfg), ctypes.byref(h))
        if st != OK:
            raise AsseError(st, "asse_init failed (see stderr)")
        self._h = h
        self.r, self.c, self.u, self.g = self.cfg.r, self.cfg.c, self.cfg.u, self.cfg.g
        self.F, self.E = 1 << self.u, 1 << self.c
        self._cap = 0

    def close(self):
        if getattr(self, "_h", None):
            self._L.asse_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st != OK:
            raise AsseError(st, self._L.asse_last_error(self._h).decode())

    @property
    def handle(self):
        return self._h

    def set_timing(self, on=True):
        self._check(self._L.asse_set_timing(self._h, 1 if on else 0))

    def set_scan_variant(self, variant):
        """0 = automatic, 1 = k_scan (direct RED.OR), 2 = k_scan_bin (shared-memory bins),
        3 = k_scan_own (packet-owned shared-memory slices; the automatic choice at C3-C5)."""
        self._check(self._L.asse_set_scan_variant(self._h, int(variant)))

    def scan_slice(self, pairs, n=None, stream=None):
        """pairs: device tensor (torch, uint32/int32, shape (n,2) or (2n,)) or a raw pointer."""
        if isinstance(pairs, int):
            ptr = pairs
            assert n is not None
        else:
            ptr = pairs.data_ptr()
            if n is None:
                n = pairs.numel() // 2
        self._check(self._L.asse_scan_slice(self._h, ptr, n, stream))

    def scan_slice_host(self, pairs):
        """pairs: host numpy uint32 (n,2) or a pinned torch CPU tensor."""
        if isinstance(pairs, np.ndarray):
            assert pairs.dtype == np.uint32 and pairs.flags.c_contiguous
            ptr, n = pairs.ctypes.data, pairs.size // 2
        else:
            ptr, n = pairs.data_ptr(), pairs.numel() // 2
        self._check(self._L.asse_scan_slice_host(self._h, ptr, n))

    def _call_reports(self, fn, *args):
        """Run an entry point that fills a report array; the returned array owns its
        memory (no copy): sized from the last call's count, retried on CAPACITY."""
        n = ctypes.c_uint32()
        cap = max(self._cap, 1024)
        while True:
            buf = np.empty(cap, dtype=REPORT_DTYPE)
            st = fn(self._h, *args[:-1], buf.ctypes.data, cap, ctypes.byref(n), args[-1])
            if st == E_CAPACITY and n.value > cap:
                cap = n.value
                self._cap = cap
                fn, args = self._L.asse_fetch_reports, (args[-1],)
                continue
            self._check(st)
            self._cap = max(self._cap, n.value)
            return buf[:n.value]

    def end_slice(self, mode=1):
        """Close the slice; returns the reports (numpy REPORT_DTYPE, ascending ip)."""
        return self._call_reports(self._L.asse_end_slice, mode)

    def end_slice_async(self, mode=1):
        """Close the slice without waiting for its results (asse_end_slice_async); the
        next slice's scan_slice may follow at once. Read them with end_slice_wait()."""
        self._check(self._L.asse_end_slice_async(self._h, mode))
        self._pend_mode = mode

    def end_slice_wait(self):
        """Reports of the pending asynchronous end_slice."""
        n = ctypes.c_uint32()
        cap = max(self._cap, 1024)
        buf = np.empty(cap, dtype=REPORT_DTYPE)
        st = self._L.asse_end_slice_wait(self._h, buf.ctypes.data, cap, ctypes.byref(n))
        if st == E_CAPACITY and n.value > cap:
            self._cap = n.value
            return self._call_reports(self._L.asse_fetch_reports, self._pend_mode)
        self._check(st)
        self._cap = max(self._cap, n.value)
        return buf[:n.value]

    def query_window(self, k_prime, mode=1):
        """Reports of the window of k_prime < k slices ending at the last closed slice."""
        return self._call_reports(self._L.asse_query_window, k_prime, mode)

    def fetch_reports(self, mode=1):
        return self._call_reports(self._L.asse_fetch_reports, mode)

    def pool(self):
        """Canonical [y][z][x][i] u16 pool (this rank's frames only with frame_shard)."""
        n = self._L.asse_pool_size(self._h)
        out = np.empty(n, dtype=np.uint16)
        self._check(self._L.asse_export_pool(self._h, out.ctypes.data, n))
        return out.reshape(self.r, -1, self.E, self.g)

    def save_state(self, path):
        self._check(self._L.asse_save_state(self._h, os.fsencode(path)))

    def load_state(self, path):
        self._check(self._L.asse_load_state(self._h, os.fsencode(path)))

    def clock(self):
        t, c0 = ctypes.c_uint64(), ctypes.c_uint32()
        self._check(self._L.asse_get_clock(self._h, ctypes.byref(t), ctypes.byref(c0)))
        return t.value, c0.value

    def keys(self):
        A, Ai, K = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        self._check(self._L.asse_get_keys(self._h, ctypes.byref(A), ctypes.byref(Ai), ctypes.byref(K)))
        return A.value, Ai.value, K.value

    def stats(self):
        s = Stats()
        self._check(self._L.asse_get_stats(self._h, ctypes.byref(s)))
        return s.as_dict()

    def stream(self):
        return self._L.asse_get_stream(self._h)

    def bitmap_bytes(self):
        return self._L.asse_bitmap_bytes(self._h)

    def merged_bytes(self):
        return self._L.asse_merged_bytes(self._h)

    def exchange_bytes(self):
        return self._L.asse_exchange_bytes(self._h)

    def attach_peers(self, touch, merged, signal=None, exchange=None, sync_mode=0):
        w = len(touch)
        arr = lambda xs: (ctypes.c_void_p * w)(*xs) if xs is not None else None
        self._check(self._L.asse_attach_peers(self._h, arr(touch), arr(merged), arr(signal),
                                              arr(exchange), sync_mode))

    def set_host_barrier(self, fn):
        """sync_mode 2: fn() is called by end_slice at each cross-rank point (after this
        rank's queued work completed) and must return once every rank has called it."""
        def _cb(_arg):
            try:
                fn()
                return 0
            except Exception:
                return 1
        self._barrier_cb = HOST_BARRIER_FN(_cb)      # kept alive with the context
        self._check(self._L.asse_set_host_barrier(self._h, self._barrier_cb, None))

    def end_slice_begin(self):
        self._check(self._L.asse_end_slice_begin(self._h))

    def merge(self):
        self._check(self._L.asse_merge(self._h))


def ipc_alloc(nbytes, device=0):
    """Zeroed device buffer for CUDA IPC sharing: returns (ptr, 64-byte handle)."""
    ptr, h = ctypes.c_void_p(), ctypes.create_string_buffer(IPC_HANDLE_BYTES)
    st = load_library().asse_ipc_alloc(device, nbytes, ctypes.byref(ptr), h)
    if st != OK:
        raise AsseError(st, "asse_ipc_alloc")
    return ptr.value, h.raw


def ipc_open(handle, device=0):
    """Map another process's asse_ipc_alloc buffer; returns the device pointer."""
    ptr = ctypes.c_void_p()
    st = load_library().asse_ipc_open(bytes(handle), device, ctypes.byref(ptr))
    if st != OK:
        raise AsseError(st, "asse_ipc_open")
    return ptr.value


def ipc_free(ptr, opened):
    st = load_library().asse_ipc_free(ptr, 1 if opened else 0)
    if st != OK:
        raise AsseError(st, "asse_ipc_free")


def selftest_barrier(world, epochs, device=0):
    """Stale reads seen by the device barrier protocol run as one cooperative kernel."""
    err = ctypes.c_uint64()
    st = load_library().asse_selftest_barrier(device, world, epochs, ctypes.byref(err))
    if st != OK:
        raise AsseError(st, "asse_selftest_barrier")
    return err.value
