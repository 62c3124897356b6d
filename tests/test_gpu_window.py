"""Parity over full windows at the production kernel instantiations.

The scan records only touches; everything the window does to the AT codes — SetAT folds,
checkAT against the cyclic ACT, preserveAT erasing ages >= k at the two swept blocks
(Alg. 2), the wrap of C0 at t = 2k — happens in k_fold. These
tests run the exact instantiations bench.py times past every one of those points and
compare the pool, CSIP, NAT and the estimates with the oracle after EVERY slice:

* C3 geometry (u8 codes, g = 512, k = 60: k_fold<1,5>, k_scan_own<1,GeoC3> chosen by the
  automatic rule at 2.6M packets/slice): 2k + 5 = 125 slices, so erasures start at t = 60
  and C0 wraps at t = 120.
* C4 shape (u16 codes, g = 512 < 2k = 600: a = 0, every AT in block 2k-1, A7; k = 300:
  k_fold<2,5>, the C4 instantiation), with c = 9, s = 7 (completeness 9 + 3*7 >= 28, 8
  duplicate positions) and 20k packets/slice to bound the oracle's time and keep the
  smaller sketch below saturation (the fold's template and its per-AT clock logic do not
  depend on c): 2k + 5 = 605 slices of the C4 mixture with its on/off DDoS spans.
* C5 at full size (100M packets/slice) through the pipelined asse_end_slice_async the
  bench uses, 3 slices.

The oracle of slice t runs in a worker thread while the device handles the same slice
(ctypes releases the GIL), so the whole-window runs stay within the suite's budget."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

from gen import PRESETS, Generator
from oracle import oracle as O
from paper_1807_01527_b200 import asse
from parity import compare_pool, compare_reports, to_device

pytestmark = pytest.mark.gpu


def _oracle_step(ora, pk):
    ora.scan(pk)
    rep = ora.end_slice(1)
    return rep, ora.pool()


def _run_window(p, gen, T, variant, expect_kernel, ctx):
    dev, ora = asse.Asse(**p), O.Oracle(**p)
    dev.set_scan_variant(variant)
    with ThreadPoolExecutor(max_workers=1) as ex:
        for t in range(T):
            pk = gen.slice(t)
            fut = ex.submit(_oracle_step, ora, pk)
            d, ptr = to_device(pk)
            dev.scan_slice(ptr, len(pk))
            rep_d = dev.end_slice(1)
            pool_d = dev.pool()
            del d
            rep_o, pool_o = fut.result()
            compare_reports(rep_d, rep_o, p["theta"], "%s t=%d" % (ctx, t))
            compare_pool(pool_d, pool_o, "%s t=%d" % (ctx, t))
    st = dev.stats()
    assert st[expect_kernel] == T, (expect_kernel, st[expect_kernel])
    assert dev.clock() == (T, T % (2 * p["k"]))
    return st


def test_full_window_c3_production_geometry(cuda_device):
    """k_scan_own (automatic choice) + k_fold<1,5> over 125 slices of C3 traffic."""
    p = dict(PRESETS["C3"])
    assert (p["k"], p["g"], p["c"], p["u"], p["s"]) == (60, 512, 12, 4, 6)
    gen = Generator("C3", N=2_600_000)
    st = _run_window(p, gen, 2 * p["k"] + 5, 0, "scan_own_launches", "C3 window")
    assert st["code_bytes"] == 1


def test_full_window_c4_shape_u16(cuda_device):
    """k_fold<2,5> (u16, a = 0) over 605 slices of the C4 mixture (DDoS bursts on/off)."""
    p = dict(PRESETS["C4"], c=9, s=7)
    assert (p["k"], p["g"]) == (300, 512)
    gen = Generator("C4", N=20_000)
    st = _run_window(p, gen, 2 * p["k"] + 5, 3, "scan_own_launches", "C4-shape window")
    assert st["code_bytes"] == 2


def test_full_size_c5_pipelined(cuda_device):
    """BASELINE C5 slices (100M packets) through the bench's pipelined step:
    scan(t) is queued behind end_slice_async(t-1) and t-1's reports are read while it
    runs; reports of every slice and the final pool equal the oracle's."""
    p = dict(PRESETS["C5"])
    dev, ora = asse.Asse(**p), O.Oracle(**p)
    gen = Generator("C5")
    T = 3
    buf = [torch.empty(2 * gen.N, dtype=torch.int32, device="cuda") for _ in range(2)]
    expect = None
    with ThreadPoolExecutor(max_workers=1) as ex:
        for t in range(T):
            b = buf[t % 2]
            gen.slice_cuda(t, b.data_ptr())
            torch.cuda.synchronize()
            host = gen.slice(t, threads=16)
            fut = ex.submit(lambda pk=host: (ora.scan(pk), ora.end_slice(1))[1])
            dev.scan_slice(b)
            if t:
                compare_reports(dev.end_slice_wait(), expect, p["theta"], "C5 async t=%d" % (t - 1))
            dev.end_slice_async(1)
            expect = fut.result()
    compare_reports(dev.end_slice_wait(), expect, p["theta"], "C5 async last")
    compare_pool(dev.pool(), ora.pool(), "C5 pipelined pool")
    assert dev.stats()["scan_own_launches"] == T
