"""ctypes wrapper of the synthetic trace generator (input infrastructure).

Presets mirror BASELINE.json.configs[0..4] (C1..C5) with the sketch geometry
reading A12 of SURVEY.md §8(c) (u=4; (c, s) = (8,7), (10,6), (12,6)).
Packets are a pure function of (preset, seed, slice t, slot j): the host fill
and the CUDA fill are bit-identical.
"""
import ctypes
import os

import numpy as np

from . import build as _build

PRESETS = {
    # name: generator preset id + sketch geometry + run shape
    "C1": dict(preset=1, seed=1, N=200_000, T=8, k=4, r=4, c=8, u=4, s=7, g=128, theta=1024.0),
    "C2": dict(preset=2, seed=2, N=2_000_000, T=30, k=10, r=4, c=10, u=4, s=6, g=256, theta=1024.0),
    "C3": dict(preset=3, seed=3, N=20_000_000, T=300, k=60, r=4, c=12, u=4, s=6, g=512, theta=1024.0),
    "C4": dict(preset=4, seed=4, N=10_000_000, T=600, k=300, r=4, c=12, u=4, s=6, g=512, theta=1024.0),
    "C5": dict(preset=5, seed=5, N=100_000_000, T=120, k=60, r=4, c=12, u=4, s=6, g=512, theta=1024.0),
    # the paper's sliding-window geometry (g=4096, r=4, c=14, u=4, k=300)
    # on the C3 traffic mixture; not a BASELINE.json config
    "PAPER": dict(preset=3, seed=3, N=20_000_000, T=600, k=300, r=4, c=14, u=4, s=6, g=4096, theta=1024.0),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        path = _build.LIB
        if not os.path.exists(path):
            _build.build()
        L = ctypes.CDLL(path)
        vp, u32, u64, i32 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
        L.gen_new.restype = vp
        L.gen_new.argtypes = [i32, u64, u64, u32]
        L.gen_free.argtypes = [vp]
        for name, rt, at in [
            ("gen_get_N", u64, [vp]), ("gen_get_T", u32, [vp]), ("gen_get_k", u32, [vp]),
            ("gen_get_n_a", u32, [vp, u32]), ("gen_plant_total", u64, [vp]),
            ("gen_planted_id", u32, [vp, u32]), ("gen_planted_m", u32, [vp, u32]),
            ("gen_victim_id", u32, [vp, u32]), ("gen_victim_onset", u32, [vp, u32]),
            ("gen_scanner_id", u32, [vp, u32]), ("gen_pool_id", u32, [vp, u32]),
        ]:
            f = getattr(L, name)
            f.restype, f.argtypes = rt, at
        L.gen_fill.restype = None
        L.gen_fill.argtypes = [vp, u32, u64, u64, u64, vp, i32]
        L.gen_cuda_fill.restype = i32
        L.gen_cuda_fill.argtypes = [vp, u32, u64, u64, u64, vp, vp]
        _lib = L
    return _lib


class Generator:
    """Seeded slice generator for preset `name` (C1..C5); N/T may be overridden."""

    def __init__(self, name, N=None, T=None, seed=None):
        p = dict(PRESETS[name])
        self.name = name
        self.params = p
        self.seed = p["seed"] if seed is None else seed
        self._h = lib().gen_new(p["preset"], self.seed, N or 0, T or 0)
        if not self._h:
            raise RuntimeError("gen_new failed")
        self.N = lib().gen_get_N(self._h)
        self.T = lib().gen_get_T(self._h)
        self.k = lib().gen_get_k(self._h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.gen_free(h)
            self._h = None

    def slice(self, t, j0=0, n=None, stride=1, threads=8):
        """Host packets of slice t: uint32 array shape (n, 2) = [aip, bip] per slot."""
        if n is None:
            n = (self.N - j0 + stride - 1) // stride
        self._check(j0, n, stride)
        out = np.empty((n, 2), dtype=np.uint32)
        lib().gen_fill(self._h, t, j0, stride, n, out.ctypes.data, threads)
        return out

    def slice_cuda(self, t, out_ptr, j0=0, n=None, stride=1, stream=0):
        """Fill n packets (slots j0 + m*stride) into device memory at out_ptr."""
        if n is None:
            n = (self.N - j0 + stride - 1) // stride
        self._check(j0, n, stride)
        rc = lib().gen_cuda_fill(self._h, t, j0, stride, n, out_ptr, stream)
        if rc != 0:
            raise RuntimeError("gen_cuda_fill failed")
        return n

    def _check(self, j0, n, stride):
        if n and (j0 + (n - 1) * stride >= self.N or stride < 1):
            raise ValueError("slots j0 + m*stride must stay below N=%d" % self.N)

    # metadata for accuracy / planted checks
    def planted(self):
        L = lib()
        n = {"C1": 4, "C2": 200}.get(self.name, 0)
        return [(L.gen_planted_id(self._h, h), L.gen_planted_m(self._h, h)) for h in range(n)]

    def victims(self):
        L = lib()
        if self.name != "C4":
            return []
        return [(L.gen_victim_id(self._h, v), L.gen_victim_onset(self._h, v)) for v in range(20)]

    def scanners(self):
        L = lib()
        if self.name not in ("C3", "C4", "C5", "PAPER"):
            return []
        return [L.gen_scanner_id(self._h, s) for s in range(50)]

    def n_a(self, a):
        return lib().gen_get_n_a(self._h, a)
