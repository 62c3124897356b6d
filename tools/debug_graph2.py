import faulthandler, sys, os
faulthandler.enable()
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), 'tests'))
import numpy as np, torch
from gen import PRESETS, Generator
from paper_1807_01527_b200 import asse
from paper_1807_01527_b200.dist import attach_local_peers, shard_slots
from parity import to_device
variant = sys.argv[1]
p = dict(PRESETS["C1"])
D = 2
ranks = [asse.Asse(**dict(p, world=D, rank=d)) for d in range(D)]
bufs = attach_local_peers(ranks)
single = asse.Asse(**p) if 'single' in variant else None
g = Generator("C1")
for t in range(5):
    pk = g.slice(t); keep = []
    for d, ctx in enumerate(ranks):
        j0, stride, n = shard_slots(len(pk), d, D)
        dp, ptr = to_device(np.ascontiguousarray(pk[j0::stride])); keep.append(dp); ctx.scan_slice(ptr, n)
    torch.cuda.synchronize()
    for ctx in ranks: ctx.merge()
    torch.cuda.synchronize()
    print(variant, t, 'end ranks', flush=True)
    reps = [ctx.end_slice(1) for ctx in ranks]
    print(variant, t, [len(r) for r in reps], flush=True)
    if single is not None:
        dfull, ptr = to_device(pk); single.scan_slice(ptr, len(pk)); rs = single.end_slice(1)
        print(variant, t, 'single', len(rs), flush=True)
