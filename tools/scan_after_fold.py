"""Does the end_slice of the previous slice slow the next binned scan? C3 workload."""
import sys
sys.path.insert(0, ".")
import torch
from gen import PRESETS, Generator
from paper_1807_01527_b200 import asse

for name in ("C3", "C5"):
    p = dict(PRESETS[name])
    ctx = asse.Asse(**p)
    g = Generator(name)
    n = g.N
    bufs = []
    for t in range(3):
        b = torch.empty(2 * n, dtype=torch.int32, device="cuda")
        g.slice_cuda(t, b.data_ptr())
        bufs.append(b)
    torch.cuda.synchronize()
    st = torch.cuda.ExternalStream(ctx.stream())
    for mode in ("scan only", "scan after end_slice"):
        ts = []
        for rep in range(8):
            if mode == "scan after end_slice":
                ctx.end_slice(0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            ctx.scan_slice(bufs[rep % 3])
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        print(name, mode, "median %.4f ms  min %.4f" % (ts[len(ts) // 2], ts[0]), flush=True)
    ctx.end_slice(0)
