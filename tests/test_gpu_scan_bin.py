"""GPU parity of the binned scan (k_scan_bin, asse_scan_bin.cuh) against the CPU oracle:
the touch bitmap is held in the SMs' shared memory, updates travel through a global
queue by owner CTA, overflowing bins fall back to a direct RED. Whatever the route, the
pool after every slice must be the oracle's bit for bit (Alg. 3; SetAT is
idempotent so the order does not matter)."""
import numpy as np
import pytest

from gen import PRESETS, Generator
from oracle import oracle as O
from paper_1807_01527_b200 import asse
from parity import step_both

pytestmark = pytest.mark.gpu


def _pair(name, variant, **over):
    p = dict(PRESETS[name], **over)
    dev = asse.Asse(**p)
    dev.set_scan_variant(variant)
    return dev, O.Oracle(**p), p


@pytest.mark.parametrize("name,N,T", [("C1", 200_000, 4), ("C2", 2_000_000, 3),
                                      ("C3", 3_000_000, 3), ("C4", 2_000_000, 3)])
def test_binned_matches_oracle(cuda_device, name, N, T):
    dev, ora, p = _pair(name, 2)
    g = Generator(name, N=N)
    for t in range(T):
        step_both(dev, ora, g.slice(t), p["theta"], "%s binned t=%d" % (name, t))
    assert dev.stats()["scan_bin_launches"] == T


def test_binned_ragged_calls_and_misalignment(cuda_device):
    """Several scan calls per slice (A34) of ragged sizes, 16-B misaligned starts (scalar
    head packet), tiny calls in which most CTAs get no tile."""
    dev, ora, p = _pair("C3", 2)
    g = Generator("C3", N=1_500_001)
    for t in range(3):
        step_both(dev, ora, g.slice(t), p["theta"], "C3 ragged t=%d" % t, split=7, offset=t % 2)
    for n in (1, 2, 3, 4097, 2048 * 148 + 5):
        pk = g.slice(3, n=n)
        step_both(dev, ora, pk, p["theta"], "C3 n=%d" % n, offset=1)


def test_binned_hot_spot_overflow(cuda_device):
    """Adversarial skew: every packet from one aip, so each row's updates of a tile land in
    one owner and overflow its CAP-entry bin; the overflow takes the direct RED route."""
    dev, ora, p = _pair("C3", 2)
    rng = np.random.default_rng(11)
    n = 2_000_000
    pk = np.stack([np.full(n, 0x0A000001, np.uint32), rng.integers(0, 2 ** 32, n, dtype=np.uint32)], 1)
    step_both(dev, ora, pk, p["theta"], "hot aip")
    # half the traffic from 3 hosts, half background
    hosts = rng.integers(0, 2 ** 32, 3, dtype=np.uint32)
    bg = Generator("C3", N=n).slice(1)
    pk2 = bg.copy()
    pk2[::2, 0] = hosts[rng.integers(0, 3, (n + 1) // 2)]
    step_both(dev, ora, pk2, p["theta"], "3 hot aips")


def test_binned_mod_p_mangle(cuda_device):
    dev, ora, p = _pair("C3", 2, mangle=1)
    g = Generator("C3", N=2_000_000)
    for t in range(2):
        step_both(dev, ora, g.slice(t), p["theta"], "C3 mod-p binned t=%d" % t)


def test_auto_variant_equals_direct_full_size(cuda_device):
    """C5 full slice (100M packets, the bench configuration): the automatic choice takes
    the binned kernel; pool and reports equal those of the direct kernel and the oracle."""
    p = dict(PRESETS["C5"])
    auto, direct = asse.Asse(**p), asse.Asse(**p)
    direct.set_scan_variant(1)
    ora = O.Oracle(**p)
    g = Generator("C5")
    pk = g.slice(0, threads=16)
    rep_a, rep_o = step_both(auto, ora, pk, p["theta"], "C5 auto")
    st = auto.stats()
    assert st["scan_bin_launches"] + st["scan_own_launches"] == 1
    import torch
    d = torch.from_numpy(pk.view(np.int32).reshape(-1)).cuda()
    direct.scan_slice(d)
    rep_d = direct.end_slice(1)
    assert direct.stats()["scan_bin_launches"] == 0
    assert (direct.pool() == auto.pool()).all()
    assert (rep_d["ip"] == rep_a["ip"]).all() and (rep_d["nat"] == rep_a["nat"]).all()


def test_variant_validation(cuda_device):
    dev = asse.Asse(**dict(PRESETS["C1"]))
    with pytest.raises(asse.AsseError):
        dev.set_scan_variant(4)
    # the paper's geometry (512 MiB touch bitmap) does not fit the shared memories
    big = asse.Asse(**dict(PRESETS["PAPER"]))
    with pytest.raises(asse.AsseError):
        big.set_scan_variant(2)
    with pytest.raises(asse.AsseError):
        big.set_scan_variant(3)
    big.set_scan_variant(0)


def test_binned_on_caller_stream_and_host_ingest(cuda_device):
    """k_scan_bin launched on a caller stream (asse_scan_slice's stream argument) and fed
    by the host double-buffered ingest (asse_scan_slice_host, 8 Mi-packet chunks)."""
    import torch
    dev, ora, p = _pair("C3", 2)
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
    assert dev.stats()["scan_bin_launches"] >= 3
