"""Pins of the oracle's reversible hash scheme RRH (§4.1)."""
import numpy as np
import pytest

from oracle import oracle as O
from asse_testutil import read_golden

PAPER_EX = dict(k=4, g=128, r=4, c=12, u=3, s=6, theta=1024.0)  # P:333 with c=12 (A11)


def test_keys_inverse_closed_form():
    """A odd and A * A^{-1} = 1 mod 2^32 (A8), checked with Python integers."""
    for seed in (1, 2, 3, 12345, 2 ** 63 + 5):
        o = O.Oracle(seed=seed, **PAPER_EX)
        A, Ai, _ = o.keys()
        assert A % 2 == 1
        assert (A * Ai) % 2 ** 32 == 1


def test_mangle_roundtrip_sample_and_exhaustive_16bit():
    """North-star check: f^{-1}(f(ip)) = ip for every IP in a sample."""
    o = O.Oracle(seed=3, **PAPER_EX)
    rng = np.random.default_rng(0)
    ips = np.concatenate([rng.integers(0, 2 ** 32, 20000, dtype=np.uint64),
                          np.arange(0, 2 ** 16, dtype=np.uint64) << np.uint64(8)])
    A, Ai, _ = o.keys()
    for ip in ips.tolist():
        h = o.mangle(ip)
        assert h == (A * ip) % 2 ** 32
        assert o.unmangle(h) == ip


def test_digest_matches_paper_worked_example():
    """x_0 = LBS[0:11], x_1 = LBS[6:17], x_3[0:10] = LBS[18:28], x_3[11] = LBS[0]."""
    rows = read_golden("rrh_paper_example.txt")
    o = O.Oracle(seed=5, **PAPER_EX)
    rng = np.random.default_rng(1)
    for h in [0xDEADBEEF, 0, 0xFFFFFFFF] + rng.integers(0, 2 ** 32, 2000).tolist():
        ip = o.unmangle(int(h))
        z, x = o.digest(ip)
        lbs = int(h) >> 3
        assert z == int(h) & 7
        for row, lo, hi, clo, chi in (map(int, r) for r in rows):
            n = hi - lo + 1
            assert ((x[row] >> clo) & ((1 << n) - 1)) == ((lbs >> lo) & ((1 << n) - 1)), (h, row)
    # the concrete value recorded in SURVEY App. A.3 for h = 0xDEADBEEF
    z, x = o.digest(o.unmangle(0xDEADBEEF))
    assert z == 7 and (0xDEADBEEF >> 3) == 0x1BD5B7DD
    assert x == [0x7DD, 0x6DF, 0xD5B, 0xEF5]


def _duplicate_positions(c, r, s, u):
    W = 32 - u
    cover = np.zeros(W, dtype=int)
    for y in range(r):
        for j in range(c):
            cover[(s * y + j) % W] += 1
    return cover


def test_restore_roundtrip_and_duplicate_check():
    """restore(digest(ip)) = ip (P:298 'Given RRH(aip), we could restore aip');
    flipping a column bit at a duplicate position makes the tuple inconsistent
    (P:320 'we remove these column tuples'); flipping a non-duplicate bit yields
    a different, consistent LBS."""
    for geo in [PAPER_EX, dict(k=4, g=128, r=4, c=8, u=4, s=7, theta=1024.0),
                dict(k=4, g=128, r=4, c=10, u=4, s=6, theta=1024.0),
                dict(k=4, g=128, r=4, c=12, u=4, s=6, theta=1024.0),
                dict(k=4, g=128, r=4, c=14, u=4, s=6, theta=1024.0)]:
        o = O.Oracle(seed=9, **geo)
        c, r, s, u = geo["c"], geo["r"], geo["s"], geo["u"]
        W = 32 - u
        cover = _duplicate_positions(c, r, s, u)
        rng = np.random.default_rng(c)
        for ip in rng.integers(0, 2 ** 32, 3000).tolist():
            z, x = o.digest(ip)
            L = o.restore_lbs(x)
            assert L == (o.mangle(ip) >> u)
            assert o.restore_ip(L, z) == ip
            y = int(rng.integers(0, r))
            j = int(rng.integers(0, c))
            pos = (s * y + j) % W
            x2 = list(x)
            x2[y] ^= 1 << j
            L2 = o.restore_lbs(x2)
            if cover[pos] >= 2:
                assert L2 is None
            else:
                assert L2 == L ^ (1 << pos)


def test_duplicate_positions_paper_example():
    """bits 6..11 (x_0/x_1 overlap) and bit 0 (x_0/x_3 wrap) are duplicate
    positions in the example geometry (the paper's '5 to 11' reads 6..11, A11)."""
    cover = _duplicate_positions(12, 4, 6, 3)
    dup = set(np.nonzero(cover >= 2)[0].tolist())
    assert {0} | set(range(6, 12)) <= dup
    assert 5 not in dup


def test_validate_examples():
    """S:249-251 / P:315-324 completeness and redundancy attributes."""
    assert O.validate(k=300, g=4096, r=4, c=14, u=4, s=6, theta=1024.0, seed=1)[0] == 0
    rc, why = O.validate(k=4, g=128, r=2, c=4, u=3, s=4, theta=1024.0, seed=1)
    assert rc != 0 and "completeness" in why
    rc, why = O.validate(k=4, g=128, r=2, c=14, u=4, s=14, theta=1024.0, seed=1)
    assert rc != 0 and "redundancy" in why
    for name in ("C1", "C2", "C3", "C4", "C5"):
        from gen import PRESETS
        assert O.validate(**PRESETS[name])[0] == 0


def test_bh_uniform_and_deterministic():
    """BH maps bip to [0, g) (A13): chi-square over 10^6 bips, g = 4096."""
    o = O.Oracle(seed=21, k=4, g=4096, r=4, c=9, u=0, s=8, theta=1024.0)
    rng = np.random.default_rng(5)
    bips = rng.integers(0, 2 ** 32, 200000).tolist()
    idx = np.array([o.bh(b) for b in bips])
    assert idx.min() >= 0 and idx.max() < 4096
    assert all(o.bh(b) == i for b, i in zip(bips[:100], idx[:100]))
    counts = np.bincount(idx, minlength=4096)
    exp = len(bips) / 4096
    chi2 = float(((counts - exp) ** 2 / exp).sum())
    # df = 4095; mean 4095, sd ~ 90.5: accept within 5 sd
    assert abs(chi2 - 4095) < 5 * 90.5


P_MANGLE = 2 ** 32 + 15   # the smallest prime above 2^32


def test_mod_p_mangle_literal_form():
    """f(aip) = A aip mod p with p prime > 2^32,
    cycle-walked into 32 bits; checked against Python integers, A A^{-1} = 1 mod p,
    and the round trip f^{-1}(f(x)) = x (including the digest/restore path)."""
    geo = dict(PAPER_EX, mangle=1)
    for seed in (1, 7, 2 ** 40 + 3):
        o = O.Oracle(seed=seed, **geo)
        A, Ai, _ = o.keys()
        assert 1 <= A < P_MANGLE and (A * Ai) % P_MANGLE == 1
        rng = np.random.default_rng(seed)
        xs = rng.integers(0, 2 ** 32, 3000).tolist() + [0, 1, 2 ** 32 - 1]
        for x in xs:
            y = A * x % P_MANGLE
            while y >= 2 ** 32:
                y = A * y % P_MANGLE
            assert o.mangle(x) == y
            assert o.unmangle(y) == x
            z, cols = o.digest(x)
            assert o.restore_ip(o.restore_lbs(cols), z) == x
    # a value whose image lands in [2^32, p) exercises the walk: search the inverse image
    o = O.Oracle(seed=1, **geo)
    A, Ai, _ = o.keys()
    t = 2 ** 32 + 3                      # A x = t (mod p)  <=>  x = Ai t
    x = Ai * t % P_MANGLE
    if x < 2 ** 32:
        y = A * t % P_MANGLE
        while y >= 2 ** 32:
            y = A * y % P_MANGLE
        assert o.mangle(x) == y and o.unmangle(y) == x
