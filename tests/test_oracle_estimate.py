"""Pins of the oracle's estimators: Eq. 3, the super-ATV threshold
 and Eq. 5 via the Eq. 4 model it inverts."""
import math

import numpy as np
import pytest

from oracle import oracle as O


@pytest.mark.parametrize("g", [8, 128, 256, 512, 1024, 4096])
def test_threshold_is_eq3_at_theta(g):
    """|ATV|_theta = g - g e^{-theta/g} is the weight at which Eq. 3 gives theta."""
    for theta in (64.0, 1024.0, 3000.0):
        if theta / g > 20:  # g e^{-theta/g} underflows relative to g: Eq. 3 saturates
            continue
        W = O.w_theta(g, theta)
        # Eq. 3 evaluated on a real weight (UP = 0 reduces Eq. 5 to Eq. 3, below)
        assert math.isclose(O.eq5_real(W, 0.0, g), theta, rel_tol=1e-8)
    assert O.eq3(0, g) == 0.0


def test_eq5_reduces_to_eq3_when_up_zero():
    for g in (128, 4096):
        for w in range(0, g, max(1, g // 37)):
            assert O.eq5(w, 0.0, g) == O.eq3(w, g)


@pytest.mark.parametrize("n,up", [(100, 0.01), (1000, 0.1), (5000, 0.3), (20000, 0.05),
                                  (1024, 0.0)])
def test_eq5_inverts_eq4_model(n, up):
    """Eq. 4: NAT = B + UP (g - B) with B = g - g e^{-n/g}; Eq. 5 must
    return n for that NAT (real-valued)."""
    g = 4096
    B = g - g * math.exp(-n / g)
    nat = B + up * (g - B)
    assert math.isclose(O.eq5_real(nat, up, g), n, rel_tol=1e-9)


def test_eq5_below_eq3_when_up_positive_and_saturation():
    """bias correction only reduces; NAT = g gives +inf (A20)."""
    g = 512
    for nat in range(0, g, 7):
        for up in (1e-4, 0.01, 0.2):
            assert O.eq5(nat, up, g) <= O.eq3(nat, g) + 1e-9
    assert O.eq5(g, 0.3, g) == math.inf


def test_linear_counting_mean_within_2pct():
    """S:151 / S:569: n = 1000 distinct peers of one host in an otherwise empty cube,
    g = 4096: the mean of Eq. 3 on its ATV weight over 100 hash seeds is within 2%."""
    n, g = 1000, 4096
    ests = []
    for seed in range(100):
        o = O.Oracle(seed=1000 + seed, k=4, g=g, r=4, c=9, u=0, s=8, theta=1024.0)
        aip = 123456789
        pairs = np.stack([np.full(n, aip, dtype=np.uint32),
                          (np.arange(n, dtype=np.uint64) * np.uint64(2654435761)) % np.uint64(2 ** 32)], 1)
        o.scan(pairs.astype(np.uint32))
        assert o.detect() == 0
        W, _, _ = o.weights()
        z, x = o.digest(aip)
        w = int(W[0, z, x[0]])
        # the ATV weight is exactly the number of distinct BH values of the peers
        assert w == len({o.bh(int(b)) for b in pairs[:, 1]})
        ests.append(O.eq3(w, g))
    assert abs(np.mean(ests) - n) / n < 0.02
