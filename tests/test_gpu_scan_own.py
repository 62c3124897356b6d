"""GPU parity of the packet-owned scan (k_scan_own, asse_scan_own.cuh) against the CPU
oracle. A packet travels once, as {f(aip), BH(bip)}, to the CTA owning (frame, word group
of its AT position), which derives the r column windows and applies the r
SetATs in shared memory; full bins fall back to direct REDs. Whatever the route, the pool
after every slice must be the oracle's bit for bit (Alg. 3; SetAT is
idempotent so the order does not matter)."""
import numpy as np
import pytest

from gen import PRESETS, Generator
from oracle import oracle as O
from paper_1807_01527_b200 import asse
from parity import step_both

pytestmark = pytest.mark.gpu


def _pair(name, **over):
    p = dict(PRESETS[name], **over)
    dev = asse.Asse(**p)
    dev.set_scan_variant(3)
    return dev, O.Oracle(**p), p


@pytest.mark.parametrize("name,N,T", [("C1", 200_000, 4), ("C2", 2_000_000, 3),
                                      ("C3", 3_000_000, 3), ("C4", 2_000_000, 3)])
def test_owned_matches_oracle(cuda_device, name, N, T):
    dev, ora, p = _pair(name)
    g = Generator(name, N=N)
    for t in range(T):
        step_both(dev, ora, g.slice(t), p["theta"], "%s owned t=%d" % (name, t))
    assert dev.stats()["scan_own_launches"] == T


def test_owned_ragged_calls_and_misalignment(cuda_device):
    """Several scan calls per slice (A34) of ragged sizes, 16-B misaligned starts (scalar
    head packet), tiny calls in which most CTAs get no tile."""
    dev, ora, p = _pair("C3")
    g = Generator("C3", N=1_500_001)
    for t in range(3):
        step_both(dev, ora, g.slice(t), p["theta"], "C3 ragged t=%d" % t, split=7, offset=t % 2)
    for n in (1, 2, 3, 4097, 2048 * 148 + 5):
        pk = g.slice(3, n=n)
        step_both(dev, ora, pk, p["theta"], "C3 n=%d" % n, offset=1)


def test_owned_hot_spot_overflow(cuda_device):
    """Adversarial skew: every packet from one aip, so every packet of a tile lands in one
    frame's NGRP owners and overflows their bins; the overflow takes the direct RED route."""
    dev, ora, p = _pair("C3")
    rng = np.random.default_rng(11)
    n = 2_000_000
    pk = np.stack([np.full(n, 0x0A000001, np.uint32), rng.integers(0, 2 ** 32, n, dtype=np.uint32)], 1)
    step_both(dev, ora, pk, p["theta"], "hot aip")
    hosts = rng.integers(0, 2 ** 32, 3, dtype=np.uint32)
    bg = Generator("C3", N=n).slice(1)
    pk2 = bg.copy()
    pk2[::2, 0] = hosts[rng.integers(0, 3, (n + 1) // 2)]
    step_both(dev, ora, pk2, p["theta"], "3 hot aips")


def test_owned_mod_p_mangle(cuda_device):
    dev, ora, p = _pair("C3", mangle=1)
    g = Generator("C3", N=2_000_000)
    for t in range(2):
        step_both(dev, ora, g.slice(t), p["theta"], "C3 mod-p owned t=%d" % t)


def test_owned_equals_binned_full_size(cuda_device):
    """C5 full slice (100M packets, the bench configuration): pools and reports of the
    packet-owned, binned and direct kernels are identical, and equal the oracle's."""
    import torch
    p = dict(PRESETS["C5"])
    own, binned, direct = asse.Asse(**p), asse.Asse(**p), asse.Asse(**p)
    own.set_scan_variant(3)
    binned.set_scan_variant(2)
    direct.set_scan_variant(1)
    ora = O.Oracle(**p)
    pk = Generator("C5").slice(0, threads=16)
    rep_own, _ = step_both(own, ora, pk, p["theta"], "C5 owned")
    d = torch.from_numpy(pk.view(np.int32).reshape(-1)).cuda()
    for other in (binned, direct):
        other.scan_slice(d)
        rep = other.end_slice(1)
        assert (other.pool() == own.pool()).all()
        assert (rep["ip"] == rep_own["ip"]).all() and (rep["nat"] == rep_own["nat"]).all()
    assert own.stats()["scan_own_launches"] == 1 and binned.stats()["scan_bin_launches"] == 1


def test_owned_on_caller_stream_and_host_ingest(cuda_device):
    import torch
    dev, ora, p = _pair("C3")
    g = Generator("C3", N=9_000_001)
    side = torch.cuda.Stream()
    pk = g.slice(0)
    with torch.cuda.stream(side):
        d = torch.from_numpy(pk.view(np.int32).reshape(-1)).to("cuda", non_blocking=False)
    dev.scan_slice(d, stream=side.cuda_stream)
    ora.scan(pk)
    rd, ro = dev.end_slice(1), ora.end_slice(1)
    assert (rd["ip"] == ro["ip"]).all() and (rd["nat"] == ro["nat"]).all()
    assert (dev.pool() == ora.pool()).all()
    pk = g.slice(1)
    dev.scan_slice_host(np.ascontiguousarray(pk))
    ora.scan(pk)
    rd, ro = dev.end_slice(1), ora.end_slice(1)
    assert (rd["ip"] == ro["ip"]).all() and (rd["nat"] == ro["nat"]).all()
    assert (dev.pool() == ora.pool()).all()
    assert dev.stats()["scan_own_launches"] >= 3


def test_owned_equals_direct_over_many_slices(cuda_device):
    """Soak: 12 consecutive C3 slices (20M packets each, ~66 rounds per launch) through the
    packet-owned and the direct kernel; pools and reports identical after every slice, so
    no round-synchronisation race shows up over ~800 rounds."""
    import torch
    p = dict(PRESETS["C3"])
    own, direct = asse.Asse(**p), asse.Asse(**p)
    own.set_scan_variant(3)
    direct.set_scan_variant(1)
    g = Generator("C3")
    for t in range(12):
        d = torch.from_numpy(g.slice(t, threads=16).view(np.int32).reshape(-1)).cuda()
        own.scan_slice(d)
        direct.scan_slice(d)
        ro, rd = own.end_slice(1), direct.end_slice(1)
        assert len(ro) == len(rd) and (ro["ip"] == rd["ip"]).all() and (ro["nat"] == rd["nat"]).all(), t
        assert (own.pool() == direct.pool()).all(), t
    assert own.stats()["scan_own_launches"] == 12 and direct.stats()["scan_own_launches"] == 0
