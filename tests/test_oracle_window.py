"""Sliding-window semantics: the exact-truth oracle against a set-based recount,
and the ASSE oracle against exact per-aip window cardinalities on tiny traces
(BASELINE.json.north_star: 'an exact per-aip hash-set sliding-window cardinality
on tiny traces')."""
import numpy as np
import pytest

from gen import PRESETS, Generator
from oracle import oracle as O


def _recount(slices, t, kp):
    win = [s for s in slices[max(0, t - kp + 1): t + 1]]
    peers = {}
    for pk in win:
        for a, b in pk.tolist():
            peers.setdefault(a, set()).add(b)
    return {a: len(v) for a, v in peers.items()}


@pytest.mark.parametrize("kp", [1, 3, 7])
def test_truth_equals_set_recount(kp):
    rng = np.random.default_rng(kp)
    T = O.Truth(kp)
    slices = []
    for t in range(20):
        n = int(rng.integers(0, 400))
        a = rng.integers(0, 12, n).astype(np.uint32) * 1000003
        b = rng.integers(0, 60, n).astype(np.uint32) + (0xFFFFFF00 if t % 5 == 0 else 0)
        pk = np.stack([a, b], 1).astype(np.uint32)
        slices.append(pk)
        T.add_slice(pk)
        exp = _recount(slices, t, kp)
        for aip, card in exp.items():
            assert T.card(aip) == card
        for aip in set(range(0, 12 * 1000003, 1000003)) - set(exp):
            assert T.card(aip) == 0
        sup, card = T.supers(10)
        assert sorted(sup.tolist()) == sorted(a for a, c in exp.items() if c >= 10)


def test_planted_c1_cardinality_exact():
    """C1 planted hosts receive 600 fresh bips per slice: window card. 600 * min(t+1, k)."""
    g = Generator("C1")
    T = O.Truth(4)
    planted = [ip for ip, _ in g.planted()]
    for t in range(6):
        T.add_slice(g.slice(t))
        for ip in planted:
            assert T.card(ip) == 600 * min(t + 1, 4)


@pytest.mark.parametrize("k,kp", [(4, 4), (6, 2), (3, 1), (300, 300)])
def test_oracle_weight_is_exact_window_on_isolated_hosts(k, kp):
    """Hosts whose RRH digests share no ATV: the weight of each host's ATV equals
    the number of distinct BH values of its exact window peers (current slice
    included, A4) at every slice end."""
    geo = dict(k=k, k_prime=kp, g=512, r=4, c=10, u=4, s=6, theta=1024.0, seed=77)
    o = O.Oracle(**geo)
    rng = np.random.default_rng(k * 10 + kp)
    hosts, used = [], set()
    while len(hosts) < 6:
        ip = int(rng.integers(0, 2 ** 32))
        z, x = o.digest(ip)
        keys = {(y, z, x[y]) for y in range(4)}
        if keys & used:
            continue
        used |= keys
        hosts.append(ip)
    slices = []
    n_slices = 12 if k < 100 else 8
    for t in range(n_slices):
        rows = []
        for h in hosts:
            m = int(rng.integers(0, 40))
            bips = rng.integers(0, 300, m).astype(np.uint32) + 7 * (t % 3)
            rows.append(np.stack([np.full(m, h, np.uint32), bips], 1))
        pk = np.concatenate(rows).astype(np.uint32)
        slices.append(pk)
        o.scan(pk)
        assert o.detect() == 0
        W, _, _ = o.weights()
        lo = max(0, t - kp + 1)
        win = np.concatenate(slices[lo:t + 1])
        for h in hosts:
            z, x = o.digest(h)
            peers = np.unique(win[win[:, 0] == h, 1])
            bh = {o.bh(int(b)) for b in peers}
            for y in range(4):
                assert W[y, z, x[y]] == len(bh), (t, h, y)
            assert o.nat(h) == len(bh)
        o.advance()


def test_detection_metrics_definition1():
    """Def. 1: FPR = N+/N, FNR = N-/N (A23)."""
    m = O.detection_metrics([1, 2, 3, 11], list(range(1, 11)))
    assert m["N"] == 10 and m["N_plus"] == 1 and m["N_minus"] == 7
    assert m["fpr"] == 0.1 and abs(m["fnr"] - 0.7) < 1e-12 and abs(m["tfr"] - 0.8) < 1e-12
