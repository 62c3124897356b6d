"""Detection accuracy of the CUDA path against exact sliding-window cardinalities
(BASELINE.json.north_star: FPR / FNR and the mean relative error must be reported;
Def. 1). These are REPORTED, not targeted (accuracy is
parity-unpinned); the assertions only check the bookkeeping and the properties the
method guarantees (planted super points with r super ATVs are found).
Set ASSE_ACCURACY_OUT=<path> to write the per-config summary as JSON."""
import json
import math
import os

import numpy as np
import pytest
import torch

from gen import PRESETS, Generator
from oracle import oracle as O
from paper_1807_01527_b200 import asse

pytestmark = pytest.mark.gpu

RESULTS = {}


def _run(name, n_slices, measure_from, N=None):
    p = dict(PRESETS[name])
    dev = asse.Asse(**p)
    g = Generator(name, N=N)
    truth = O.Truth(p["k"])
    buf = torch.empty(2 * g.N, dtype=torch.int32, device="cuda")
    per = []
    for t in range(n_slices):
        g.slice_cuda(t, buf.data_ptr())
        dev.scan_slice(buf)
        rep = dev.end_slice(0)                       # est >= theta (A21)
        torch.cuda.synchronize()
        truth.add_slice(buf.cpu().numpy().view(np.uint32).reshape(-1, 2))
        if t < measure_from:
            continue
        tips, tcard = truth.supers(p["theta"])
        m = O.detection_metrics(rep["ip"], tips)
        card = dict(zip(tips.tolist(), tcard.tolist()))
        rel = [abs(r["estimate"] - card[int(r["ip"])]) / card[int(r["ip"])]
               for r in rep if int(r["ip"]) in card and math.isfinite(r["estimate"])]
        n_sat = int(((rep["flags"] & 1) != 0).sum())
        per.append(dict(t=t, N=m["N"], detected=len(rep), N_plus=m["N_plus"], N_minus=m["N_minus"],
                        fpr=m["fpr"], fnr=m["fnr"], tfr=m["tfr"], mre=float(np.mean(rel)) if rel else None,
                        saturated=n_sat, csip=dev.stats()["last_n_candidates"]))
    mean = lambda k: float(np.mean([x[k] for x in per if x[k] is not None])) if any(
        x[k] is not None for x in per) else None
    summary = dict(config=name, packets_per_slice=g.N, slices=n_slices, windows_measured=len(per),
                   true_super_points=mean("N"), detected=mean("detected"), csip=mean("csip"),
                   saturated=mean("saturated"), fpr=mean("fpr"), fnr=mean("fnr"), tfr=mean("tfr"),
                   mre=mean("mre"), per_window=per)
    RESULTS[name] = summary
    out = os.environ.get("ASSE_ACCURACY_OUT")
    if out:
        with open(out, "w") as f:
            json.dump(RESULTS, f, indent=1)
    return summary, g


def test_accuracy_c1(cuda_device):
    s, g = _run("C1", 8, 3)
    assert s["true_super_points"] >= 4
    # g = 128 < g ln g: W_theta = 128, super ATVs must be saturated; hosts just above
    # theta can miss (SURVEY §8(d) expects FNR ~ 0 and FPR ~ 89 here)
    assert s["fnr"] < 0.05 and s["fpr"] > 1


def test_accuracy_c2(cuda_device):
    s, g = _run("C2", 30, 9)
    assert s["true_super_points"] > 100 and s["fnr"] < 0.5


def test_accuracy_c3_reduced(cuda_device):
    """C3 traffic at 5M packets/slice through its first full window (the BASELINE-size
    C3/C4/C5 and g-sweep reports: tools/accuracy.py -> profiles/accuracy_r02.json)."""
    s, g = _run("C3", 62, 59, N=5_000_000)
    assert s["true_super_points"] > 100 and s["fnr"] < 0.5
