"""Pins of the oracle's restore (Alg. 4) and NAT (Alg. 5)
against brute force and invariants, on the C1 trace (BASELINE.json.configs[0])."""
import numpy as np
import pytest

from gen import PRESETS, Generator
from oracle import oracle as O


def _active_pool(pool, C0, k, kp, g):
    """Activity of every AT from an exported pool: last set within the latest k'
    slices, with the block ACT (C0 + block) mod 2k of P:256."""
    two_k = 2 * k
    a = g // two_k
    i = np.arange(g)
    blk = np.minimum(i // a, two_k - 1) if a > 0 else np.full(g, two_k - 1)
    act = (C0 + blk) % two_k
    v = pool.astype(np.int64)
    age = (act - v) % two_k
    return (v != two_k) & (age <= kp - 1)


def _brute_csip(sup, A, c, s, u, r):
    """All ip in [0, 2^32) whose r ATVs are super (the plain definition, A16):
    enumerate every LBS whose row-0 column is super (a necessary condition),
    then test rows 1..r-1; ip = A^{-1} ((LBS << u) | z)."""
    W = 32 - u
    Ainv = pow(A, -1, 2 ** 32)
    cmask = (1 << c) - 1
    free = np.arange(1 << (W - c), dtype=np.uint64) << np.uint64(c)
    out = []
    for z in range(1 << u):
        for x0 in np.nonzero(sup[0, z])[0]:
            L = free | np.uint64(x0)
            D = L | (L << np.uint64(W))
            ok = np.ones(L.shape, dtype=bool)
            for y in range(1, r):
                xy = (D >> np.uint64(s * y)) & np.uint64(cmask)
                ok &= sup[y, z][xy.astype(np.int64)].astype(bool)
            Ls = L[ok]
            ips = ((Ls << np.uint64(u)) | np.uint64(z)) * np.uint64(Ainv) % np.uint64(2 ** 32)
            out.append(ips)
    return np.sort(np.concatenate(out)).astype(np.uint32) if out else np.zeros(0, np.uint32)


@pytest.fixture(scope="module")
def c1_run():
    p = dict(PRESETS["C1"])
    o = O.Oracle(**p)
    g = Generator("C1")
    slices = []
    for t in range(p["T"]):
        pk = g.slice(t)
        o.scan(pk)
        assert o.detect() == 0
        W, aat, sup = o.weights()
        slices.append(dict(t=t, pk=pk, pool=o.pool().copy(), W=W, aat=aat, sup=sup,
                           rep=o.reports(), C0=o.C0))
        o.advance()
    return p, o, g, slices


def test_weights_match_recount(c1_run):
    p, o, _, slices = c1_run
    for S in slices:
        act = _active_pool(S["pool"], S["C0"], p["k"], p["k"], p["g"])
        W = act.sum(-1)
        assert (W == S["W"]).all()
        assert (W.sum(-1) == S["aat"]).all()
        thr = O.w_theta(p["g"], p["theta"])
        assert ((W >= thr) == S["sup"].astype(bool)).all()


@pytest.mark.parametrize("t", [1, 3, 7])
def test_csip_equals_brute_force(c1_run, t):
    p, o, _, slices = c1_run
    S = slices[t]
    A, _, _ = o.keys()
    brute = _brute_csip(S["sup"], A, p["c"], p["s"], p["u"], p["r"])
    rep = S["rep"]
    assert len(rep) == len(brute) > 0
    assert (rep["ip"] == brute).all()            # ascending ip (A24), no duplicates


def test_planted_super_points_restored(c1_run):
    """a host whose r ATVs are all super is in CSIP; the 4 planted C1 hosts
    (600 fresh peers per slice) are super points from slice 1 on."""
    p, o, g, slices = c1_run
    planted = [ip for ip, _ in g.planted()]
    for S in slices[1:]:
        ips = set(S["rep"]["ip"].tolist())
        for ip in planted:
            assert ip in ips


def test_nat_invariants(c1_run):
    """min_y w_y >= NAT >= |{BH(bip) : bip a true in-window peer}|,
    and NAT equals the recount of ATs active in all r ATVs (Alg. 5)."""
    p, o, g, slices = c1_run
    k = p["k"]
    for S in slices[2:5]:
        t = S["t"]
        win = np.concatenate([slices[q]["pk"] for q in range(max(0, t - k + 1), t + 1)])
        act = _active_pool(S["pool"], S["C0"], k, k, p["g"])
        rep = S["rep"]
        pick = rep[np.linspace(0, len(rep) - 1, 40).astype(int)]
        for R in pick:
            z, x = o.digest(int(R["ip"]))
            rows = np.stack([act[y, z, x[y]] for y in range(p["r"])])
            nat = int(rows.all(0).sum())
            assert nat == R["nat"]
            assert min(int(S["W"][y, z, x[y]]) for y in range(p["r"])) >= nat
            peers = np.unique(win[win[:, 0] == R["ip"], 1])
            assert nat >= len({o.bh(int(b)) for b in peers})
            # Eq. 4/5 inputs: UP from AAT
            up = 1.0
            for y in range(p["r"]):
                up *= float(S["aat"][y, z]) / (p["g"] * 2 ** p["c"])
            assert R["estimate"] == O.eq5(nat, up, p["g"])


def test_overflow_is_reported():
    p = dict(PRESETS["C1"], max_candidates=10)
    o = O.Oracle(**p)
    o.scan(Generator("C1").slice(0))
    o.scan(Generator("C1").slice(1))
    assert o.detect() == -4
