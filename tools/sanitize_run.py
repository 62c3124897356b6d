"""Small end-to-end run of the library for compute-sanitizer (memcheck / racecheck):
C1 slices, odd / misaligned / empty scans, window queries, host ingest, a g=1024
geometry and virtual multi-rank merge."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gen import PRESETS, Generator  # noqa: E402
from paper_1807_01527_b200 import asse  # noqa: E402
from paper_1807_01527_b200.dist import attach_local_peers, shard_slots  # noqa: E402


def dev(pk):
    return torch.from_numpy(np.ascontiguousarray(pk).view(np.int32).reshape(-1)).cuda()


p = dict(PRESETS["C1"])
a = asse.Asse(**p)
g = Generator("C1")
for t in range(4):
    pk = g.slice(t)
    d = dev(pk)
    a.scan_slice(d.data_ptr() + 8, len(pk) - 1)   # misaligned, odd
    a.scan_slice(d.data_ptr(), 1)
    r = a.end_slice(1 if t % 2 else 0)
    print("C1", t, len(r), flush=True)
a.scan_slice_host(np.ascontiguousarray(g.slice(5)))
a.end_slice(1)
a.end_slice(1)                                     # empty slice
print("query", len(a.query_window(2)), flush=True)
b = asse.Asse(k=10, r=4, c=8, u=4, s=7, g=1024, theta=1024.0, seed=3)
g2 = Generator("C2", N=200_000)
for t in range(3):
    d = dev(g2.slice(t))
    b.scan_slice(d)
    print("g1024", t, len(b.end_slice(1)), flush=True)
D = 2
ranks = [asse.Asse(**dict(p, world=D, rank=r)) for r in range(D)]
bufs = attach_local_peers(ranks)
for t in range(2):
    pk = g.slice(t)
    keep = []
    for r, ctx in enumerate(ranks):
        j0, stride, n = shard_slots(len(pk), r, D)
        keep.append(dev(pk[j0::stride]))
        ctx.scan_slice(keep[-1])
    torch.cuda.synchronize()
    for ctx in ranks:
        ctx.merge()
    torch.cuda.synchronize()
    print("ranks", t, [len(ctx.end_slice(1)) for ctx in ranks], flush=True)
torch.cuda.synchronize()
print("sanitize run ok", flush=True)

# binned scan (k_scan_bin) on the C3 geometry: forced variant, ragged + misaligned calls,
# pipelined end_slice
p3 = dict(PRESETS["C3"])
b = asse.Asse(**p3)
b.set_scan_variant(2)
g3 = Generator("C3", N=400_001)
for t in range(3):
    pk = g3.slice(t)
    d = dev(pk)
    b.scan_slice(d.data_ptr() + 8, len(pk) - 1)
    b.scan_slice(d.data_ptr(), 3)
    if t:
        print("C3 bin", t - 1, len(b.end_slice_wait()), flush=True)
    b.end_slice_async(1)
    torch.cuda.synchronize()
print("C3 bin last", len(b.end_slice_wait()), flush=True)

# packet-owned scan (k_scan_own) on the C3 geometry (constant-folded instantiation) and on
# C2 (runtime geometry): ragged + misaligned calls, a hot-spot overflow slice
for name in ("C3", "C2"):
    po = dict(PRESETS[name])
    o = asse.Asse(**po)
    o.set_scan_variant(3)
    go = Generator(name, N=400_001)
    for t in range(2):
        pk = go.slice(t)
        d = dev(pk)
        o.scan_slice(d.data_ptr() + 8, len(pk) - 1)
        o.scan_slice(d.data_ptr(), 3)
        print(name, "own", t, len(o.end_slice(1)), flush=True)
    hot = np.stack([np.full(300_000, 0x0A000001, np.uint32),
                    np.random.default_rng(1).integers(0, 2 ** 32, 300_000, dtype=np.uint32)], 1)
    d = dev(hot)
    o.scan_slice(d)
    print(name, "own hot", len(o.end_slice(1)), flush=True)
torch.cuda.synchronize()
print("sanitize run (k_scan_own) ok", flush=True)
