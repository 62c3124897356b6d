"""Per-CTA timeline of k_restore (tools only): run with ASSE_LIB pointing at a build with
-D ASSE_RESTORE_PROF=1 (python tools/sweep.py build rprof -D ASSE_RESTORE_PROF=1). Marks:
0 entry, 1 after griddepcontrol.wait, 2 after the prologue barrier, 3-6 after rows 0-3,
7 end; printed as min / median / max over CTAs, relative to the earliest entry (us)."""
import ctypes
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from gen import PRESETS, Generator
from paper_1807_01527_b200 import asse

w = sys.argv[1] if len(sys.argv) > 1 else "C3"
p = dict(PRESETS[w])
ctx = asse.Asse(**p)
g = Generator(w)
buf = torch.empty(2 * g.N, dtype=torch.int32, device="cuda")
lib = asse.load_library()
fn = lib.asse_debug_restore_prof
fn.argtypes = [ctypes.c_void_p, ctypes.c_uint]
for t in range(8):
    g.slice_cuda(t, buf.data_ptr())
    torch.cuda.synchronize()
    ctx.scan_slice(buf)
    ctx.end_slice(1)
    torch.cuda.synchronize()
    h = np.zeros((4096, 8), np.uint64)
    fn(h.ctypes.data, 4096)
    n = int((h[:, 0] > 0).sum())
    h = h[:n].astype(np.float64)
    t0 = h[:, 0].min()
    rel = (h - t0) / 1e3
    if t >= 5:
        print(w, "slice", t, "CTAs", n, " ".join("m%d %.2f/%.2f/%.2f" % (k, rel[:, k].min(), np.median(rel[:, k]), rel[:, k].max())
                                            for k in range(8)))
