"""Fixed vs per-round cost of k_scan_bin (argv[1] = 2) or k_scan_own (3): time scans of R rounds (R * 148 * 2048 packets of
the C5 mixture) for several R and fit t = a + b R."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from gen import PRESETS, Generator
from paper_1807_01527_b200 import asse

p = dict(PRESETS["C5"])
ctx = asse.Asse(**p)
ctx.set_scan_variant(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
G = torch.cuda.get_device_properties(0).multi_processor_count
g = Generator("C5")
buf = torch.empty(2 * 100_000_000, dtype=torch.int32, device="cuda")
g.slice_cuda(0, buf.data_ptr())
torch.cuda.synchronize()
st = torch.cuda.ExternalStream(ctx.stream())
res = []
for R in (8, 12, 16, 24, 32, 48, 64, 128, 256, 329):
    n = min(100_000_000, R * G * 2048)
    ts = []
    for rep in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        ctx.scan_slice(buf, n)
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ctx.end_slice(0)
    t = sorted(ts)[len(ts) // 2]
    res.append((R, n, t))
    print("rounds %4d packets %10d  %.4f ms  %.2f Gpps" % (R, n, t, n / t / 1e6), flush=True)
R = np.array([r for r, _, _ in res], float)
T = np.array([t for _, _, t in res])
b, a = np.polyfit(R, T, 1)
print("fit: fixed %.4f ms + %.5f ms/round (%.1f Gpps steady)" % (a, b, G * 2048 / b / 1e6))
