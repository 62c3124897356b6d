"""ctypes binding of the CPU oracle (oracle/asse_oracle.c) and the exact-truth
oracle (oracle/truth.c).

TEST INFRASTRUCTURE. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module. The product path
(paper_1807_01527_b200) never does, and the oracle never imports it.
"""
import ctypes
import os

import numpy as np

from . import build as _build

REPORT_DTYPE = np.dtype([("ip", "<u4"), ("nat", "<u4"), ("estimate", "<f8"),
                         ("flags", "<u4"), ("pad", "<u4")])
SATURATED, ABOVE_THETA = 1, 2


class _Params(ctypes.Structure):
    _fields_ = [("k", ctypes.c_uint32), ("k_prime", ctypes.c_uint32), ("r", ctypes.c_uint32),
                ("c", ctypes.c_uint32), ("u", ctypes.c_uint32), ("s", ctypes.c_uint32),
                ("g", ctypes.c_uint32), ("theta", ctypes.c_double), ("seed", ctypes.c_uint64),
                ("max_candidates", ctypes.c_uint32), ("mangle", ctypes.c_uint32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        path = _build.build()
        L = ctypes.CDLL(path)
        vp, u32, u64, i32, dbl = (ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64,
                                  ctypes.c_int, ctypes.c_double)
        P = ctypes.POINTER(_Params)
        sigs = {
            "oracle_validate": (i32, [P, ctypes.c_char_p, ctypes.c_size_t]),
            "oracle_new": (vp, [P, ctypes.c_char_p, ctypes.c_size_t]),
            "oracle_free": (None, [vp]),
            "oracle_check_at": (i32, [u32, u32, u32, u32]),
            "oracle_preserve_at": (u32, [u32, u32, u32]),
            "oracle_eq3": (dbl, [u32, u32]),
            "oracle_eq5": (dbl, [u32, dbl, u32]),
            "oracle_eq5_real": (dbl, [dbl, dbl, u32]),
            "oracle_w_theta": (dbl, [u32, dbl]),
            "oracle_block": (u32, [vp, u32]),
            "oracle_act": (u32, [vp, u32]),
            "oracle_mangle": (u32, [vp, u32]),
            "oracle_unmangle": (u32, [vp, u32]),
            "oracle_digest": (None, [vp, u32, vp, vp]),
            "oracle_bh": (u32, [vp, u32]),
            "oracle_restore_lbs": (i32, [vp, vp, vp]),
            "oracle_restore_ip": (u32, [vp, u32, u32]),
            "oracle_keys": (None, [vp, vp, vp, vp]),
            "oracle_blocks": (None, [vp, vp, vp]),
            "oracle_C0": (u32, [vp]),
            "oracle_slice": (u64, [vp]),
            "oracle_pool_size": (u64, [vp]),
            "oracle_touch": (None, [vp, u32, u32, u32, u32]),
            "oracle_scan": (None, [vp, vp, u64]),
            "oracle_scan_mt": (None, [vp, vp, u64, i32]),
            "oracle_omp_threads": (i32, []),
            "oracle_nat": (u32, [vp, u32]),
            "oracle_detect": (i32, [vp]),
            "oracle_advance": (None, [vp]),
            "oracle_end_slice": (i32, [vp, i32, vp, u32, vp]),
            "oracle_export_pool": (None, [vp, vp]),
            "oracle_import_pool": (None, [vp, vp]),
            "oracle_weights": (None, [vp, vp, vp, vp]),
            "oracle_n_reports": (u32, [vp]),
            "oracle_reports": (None, [vp, vp]),
            "oracle_combine_min_age": (None, [vp, vp, u32, vp]),
            "truth_new": (vp, [u32]),
            "truth_free": (None, [vp]),
            "truth_begin_slice": (None, [vp]),
            "truth_add": (None, [vp, vp, u64]),
            "truth_card": (u32, [vp, u32]),
            "truth_supers": (u64, [vp, u32, vp, vp, u64]),
        }
        for name, (rt, at) in sigs.items():
            f = getattr(L, name)
            f.restype, f.argtypes = rt, at
        _lib = L
    return _lib


def check_at(at, act, k, kp):
    return bool(lib().oracle_check_at(at, act, k, kp))


def preserve_at(at, act, k):
    return lib().oracle_preserve_at(at, act, k)


def eq3(w, g):
    return lib().oracle_eq3(w, g)


def eq5(nat, up, g):
    return lib().oracle_eq5(nat, up, g)


def eq5_real(nat, up, g):
    return lib().oracle_eq5_real(nat, up, g)


def w_theta(g, theta):
    return lib().oracle_w_theta(g, theta)


def _params(k, r, c, u, s, g, theta, seed, k_prime=0, max_candidates=1 << 24, mangle=0, **_):
    return _Params(k, k_prime or k, r, c, u, s, g, float(theta), seed, max_candidates, mangle)


def validate(**kw):
    why = ctypes.create_string_buffer(256)
    p = _params(**kw)
    rc = lib().oracle_validate(ctypes.byref(p), why, 256)
    return rc, why.value.decode()


class Oracle:
    """ASSE CPU oracle; keyword geometry as in gen.PRESETS (k, r, c, u, s, g, theta, seed)."""

    def __init__(self, **kw):
        self.kw = dict(kw)
        self.p = _params(**kw)
        why = ctypes.create_string_buffer(256)
        self._h = lib().oracle_new(ctypes.byref(self.p), why, 256)
        if not self._h:
            raise ValueError("oracle_new: " + why.value.decode())
        self.r, self.c, self.u, self.g, self.k = self.p.r, self.p.c, self.p.u, self.p.g, self.p.k
        self.F, self.E = 1 << self.u, 1 << self.c

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.oracle_free(h)
            self._h = None

    # ---- keys / hashing
    def keys(self):
        A, Ai, K = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        lib().oracle_keys(self._h, ctypes.byref(A), ctypes.byref(Ai), ctypes.byref(K))
        return A.value, Ai.value, K.value

    def blocks(self):
        a, b = ctypes.c_uint32(), ctypes.c_uint32()
        lib().oracle_blocks(self._h, ctypes.byref(a), ctypes.byref(b))
        return a.value, b.value

    def mangle(self, ip):
        return lib().oracle_mangle(self._h, ip)

    def unmangle(self, h):
        return lib().oracle_unmangle(self._h, h)

    def digest(self, ip):
        z = ctypes.c_uint32()
        x = (ctypes.c_uint32 * self.r)()
        lib().oracle_digest(self._h, ip, ctypes.byref(z), x)
        return z.value, list(x)

    def bh(self, bip):
        return lib().oracle_bh(self._h, bip)

    def restore_lbs(self, xs):
        x = (ctypes.c_uint32 * self.r)(*xs)
        L = ctypes.c_uint32()
        ok = lib().oracle_restore_lbs(self._h, x, ctypes.byref(L))
        return L.value if ok else None

    def restore_ip(self, lbs, z):
        return lib().oracle_restore_ip(self._h, lbs, z)

    def block(self, i):
        return lib().oracle_block(self._h, i)

    def act(self, i):
        return lib().oracle_act(self._h, i)

    @property
    def C0(self):
        return lib().oracle_C0(self._h)

    @property
    def t(self):
        return lib().oracle_slice(self._h)

    # ---- per-slice operation
    def touch(self, y, z, x, i):
        lib().oracle_touch(self._h, y, z, x, i)

    def scan(self, pairs):
        pairs = np.ascontiguousarray(pairs, dtype=np.uint32)
        lib().oracle_scan(self._h, pairs.ctypes.data, pairs.size // 2)

    def scan_mt(self, pairs, nthreads=0):
        """All-core variant of scan (bench.py's optional CPU baseline only; same pool)."""
        pairs = np.ascontiguousarray(pairs, dtype=np.uint32)
        lib().oracle_scan_mt(self._h, pairs.ctypes.data, pairs.size // 2, int(nthreads))

    def detect(self):
        return lib().oracle_detect(self._h)

    def advance(self):
        lib().oracle_advance(self._h)

    def nat(self, ip):
        return lib().oracle_nat(self._h, ip)

    def reports(self):
        n = lib().oracle_n_reports(self._h)
        out = np.zeros(n, dtype=REPORT_DTYPE)
        if n:
            lib().oracle_reports(self._h, out.ctypes.data)
        return out

    def end_slice(self, mode=1):
        """Detect at t, return reports (mode 0: est >= theta; 1: all CSIP), advance to t+1."""
        n = ctypes.c_uint32()
        rc = lib().oracle_end_slice(self._h, mode, None, 0, ctypes.byref(n))
        # reports of the detect step are still held by the oracle
        rep = self.reports()
        if rc not in (0, -3):
            raise OverflowError("oracle_end_slice status %d" % rc)
        if mode == 0:
            rep = rep[(rep["flags"] & ABOVE_THETA) != 0]
        return rep

    def weights(self):
        n_atv = self.r * self.F * self.E
        w = np.zeros(n_atv, dtype=np.uint32)
        aat = np.zeros(self.r * self.F, dtype=np.uint64)
        sup = np.zeros(n_atv, dtype=np.uint8)
        lib().oracle_weights(self._h, w.ctypes.data, aat.ctypes.data, sup.ctypes.data)
        return (w.reshape(self.r, self.F, self.E), aat.reshape(self.r, self.F),
                sup.reshape(self.r, self.F, self.E))

    def pool(self):
        n = lib().oracle_pool_size(self._h)
        out = np.empty(n, dtype=np.uint16)
        lib().oracle_export_pool(self._h, out.ctypes.data)
        return out.reshape(self.r, self.F, self.E, self.g)

    def set_pool(self, pool):
        pool = np.ascontiguousarray(pool, dtype=np.uint16)
        lib().oracle_import_pool(self._h, pool.ctypes.data)

    def combine_min_age(self, pools):
        arrs = [np.ascontiguousarray(p, dtype=np.uint16) for p in pools]
        ptrs = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
        out = np.empty_like(arrs[0])
        lib().oracle_combine_min_age(self._h, ptrs, len(arrs), out.ctypes.data)
        return out


class Truth:
    """Exact per-aip sliding-window distinct-peer counts over the last k' slices."""

    def __init__(self, k_prime):
        self._h = lib().truth_new(k_prime)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.truth_free(h)
            self._h = None

    def add_slice(self, pairs):
        pairs = np.ascontiguousarray(pairs, dtype=np.uint32)
        lib().truth_begin_slice(self._h)
        lib().truth_add(self._h, pairs.ctypes.data, pairs.size // 2)

    def card(self, aip):
        return lib().truth_card(self._h, int(aip))

    def supers(self, theta):
        n = lib().truth_supers(self._h, int(theta), None, None, 0)
        ips = np.zeros(n, dtype=np.uint32)
        card = np.zeros(n, dtype=np.uint32)
        if n:
            lib().truth_supers(self._h, int(theta), ips.ctypes.data, card.ctypes.data, n)
        order = np.argsort(ips)
        return ips[order], card[order]


def detection_metrics(detected_ips, true_ips):
    """Definition 1: FPR = N+/N, FNR = N-/N, TFR = FPR + FNR (A23)."""
    det, tru = set(int(x) for x in detected_ips), set(int(x) for x in true_ips)
    N = len(tru)
    n_plus = len(det - tru)
    n_minus = len(tru - det)
    if N == 0:
        return dict(N=0, N_plus=n_plus, N_minus=n_minus, fpr=None, fnr=None, tfr=None)
    return dict(N=N, N_plus=n_plus, N_minus=n_minus, fpr=n_plus / N, fnr=n_minus / N,
                tfr=(n_plus + n_minus) / N)
