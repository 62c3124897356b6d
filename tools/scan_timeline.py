import sys, os
sys.path.insert(0, ".")
import torch
from gen import PRESETS, Generator
from paper_1807_01527_b200 import asse
p = dict(PRESETS["C5"])
ctx = asse.Asse(**p)
ctx.set_scan_variant(3)
g = Generator("C5")
buf = torch.empty(2 * 100_000_000, dtype=torch.int32, device="cuda")
g.slice_cuda(0, buf.data_ptr())
torch.cuda.synchronize()
st = torch.cuda.ExternalStream(ctx.stream())
for n in (10_000_000, 20_000_000, 100_000_000):
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); ctx.scan_slice(buf, n); e1.record(st); torch.cuda.synchronize()
        print("n", n, "ms", e0.elapsed_time(e1), file=sys.stderr, flush=True)
        ctx.end_slice(0)
