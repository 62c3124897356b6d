import faulthandler, sys, os
faulthandler.enable()
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), 'tests'))
import numpy as np, torch
from gen import PRESETS, Generator
from paper_1807_01527_b200 import asse
from paper_1807_01527_b200.dist import attach_local_peers, shard_slots
from parity import to_device
p = dict(PRESETS["C1"])
print("single", flush=True)
a = asse.Asse(**p); g = Generator("C1")
for t in range(3):
    d, ptr = to_device(g.slice(t)); a.scan_slice(ptr, g.N); r = a.end_slice(1); print(t, len(r), flush=True)
a.set_timing(True)
d, ptr = to_device(g.slice(3)); a.scan_slice(ptr, g.N); r = a.end_slice(1); print('timed', len(r), a.stats()['last_end_slice_ms'], flush=True)
print("multi", flush=True)
D = 2
ranks = [asse.Asse(**dict(p, world=D, rank=d)) for d in range(D)]
bufs = attach_local_peers(ranks)
print("attached", flush=True)
for t in range(3):
    pk = g.slice(t); keep = []
    for d, ctx in enumerate(ranks):
        j0, stride, n = shard_slots(len(pk), d, D)
        dp, ptr = to_device(np.ascontiguousarray(pk[j0::stride])); keep.append(dp); ctx.scan_slice(ptr, n)
    torch.cuda.synchronize()
    for ctx in ranks: ctx.merge()
    torch.cuda.synchronize(); print('merged', flush=True)
    reps = [ctx.end_slice(1) for ctx in ranks]
    print(t, [len(r) for r in reps], flush=True)
