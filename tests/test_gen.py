"""The synthetic trace generator (input infrastructure)."""
import numpy as np
import pytest

from gen import Generator
from oracle import oracle as O


def test_deterministic_and_shardable():
    for name in ("C1", "C2", "C3", "C4"):
        g = Generator(name)
        a = g.slice(3, n=50000)
        b = Generator(name).slice(3, n=50000)
        assert (a == b).all()
        # round-robin shard (packet j -> rank j mod D, BASELINE.json.configs[4]) is a sub-sample
        D = 4
        for rank in range(D):
            s = g.slice(3, j0=rank, stride=D, n=5000)
            assert (s == a[rank::D][:5000]).all()
        assert not (g.slice(4, n=1000) == a[:1000]).all()
        with pytest.raises(ValueError):
            g.slice(0, j0=g.N - 1, n=2)


def test_c1_shape():
    g = Generator("C1")
    pk = g.slice(0)
    assert pk.shape == (200000, 2)
    planted = dict(g.planted())
    for ip, m in planted.items():
        sel = pk[pk[:, 0] == ip]
        assert len(sel) == m == 600 and len(np.unique(sel[:, 1])) == 600
    bg = pk[~np.isin(pk[:, 0], list(planted))]
    assert len(np.unique(bg[:, 0])) <= 16384


def test_c2_planted_window_cardinality():
    """200 planted hosts, window cardinality ~ n_p in [512, 65536] (k = 10 slices)."""
    g = Generator("C2", N=400000)
    T = O.Truth(10)
    for t in range(10):
        T.add_slice(g.slice(t))
    cards = [T.card(ip) for ip, m in g.planted()]
    ms = [m for _, m in g.planted()]
    assert cards == [10 * m for m in ms]
    assert 500 <= min(cards) and max(cards) <= 65540


def test_c3_mixture_fractions():
    g = Generator("C3", N=400000)
    pk = g.slice(0)
    scanners = set(g.scanners())
    is_scan = np.isin(pk[:, 0], list(scanners))
    assert abs(is_scan.mean() - 0.05 * 1.25) < 0.01  # 5% fresh + copies made by duplicates
    key = pk[:, 0].astype(np.uint64) << np.uint64(32) | pk[:, 1]
    dup = 1 - len(np.unique(key)) / len(key)
    assert 0.18 < dup < 0.30


def test_c4_victims_switch_on_and_off():
    g = Generator("C4", N=200000)
    for ip, on in g.victims()[:5]:
        for t in (on - 1, on, on + 49, on + 50):
            if t < 0:
                continue
            n = int((g.slice(t)[:, 0] == ip).sum())
            assert (n == 1000) == (on <= t < on + 50), (ip, on, t, n)
