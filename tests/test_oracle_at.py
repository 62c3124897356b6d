"""Pins of the oracle's AT / ATV layer (§3) against
things other than itself: the paper's k=9 worked example, a hand-worked table,
and an exact "last set within the latest k' slices" model."""
import numpy as np
import pytest

from oracle import oracle as O
from asse_testutil import read_golden

# Small valid cubes (completeness + redundancy) used to host single ATVs.
TINY = dict(r=4, c=10, u=2, s=10, theta=1024.0, seed=7)
MICRO = dict(r=16, c=3, u=0, s=3, theta=1024.0, seed=11)   # 128 ATVs, F = 1


def test_preserve_paper_k9_example():
    """act 0 -> values 0..9 become 18; act 9 -> 0 and 9..17 become 18."""
    rows = read_golden("at_k9_preserve.txt")
    assert len(rows) == 38
    for act, before, after in rows:
        assert O.preserve_at(int(before), int(act), 9) == int(after), (act, before)
    # every other act leaves values untouched (Alg. 2, act mod k != 0)
    for act in range(1, 18):
        if act == 9:
            continue
        for v in range(19):
            assert O.preserve_at(v, act, 9) == v


def test_check_at_reading_examples():
    """Alg. 1 on the inactive sentinel and distance wrap ('set one wrap ago')."""
    assert not O.check_at(600, 5, 300, 300)
    assert O.check_at(3, 5, 300, 300)            # dis 2
    assert not O.check_at(5, 10, 300, 5)         # dis 5 > 4
    assert not O.check_at(7, 5, 300, 300)        # dis 598


def _expected_after(last, t_end, k, g):
    """Exact model of an AT's stored value at time t_end (preserve applied at every
    slice start s <= t_end): preserveAT erases exactly the values set >= k slices
    before a preserve point of their block (P:243 'labeled inactive when the
    distance is bigger than k'; preserve points are the slices whose block ACT is
    0 or k). Returns (value array, active-age array)."""
    two_k = 2 * k
    a = g // two_k
    vals = np.full(g, two_k, dtype=np.int64)
    for i in range(g):
        if last[i] < 0:
            continue
        b = min(i // a, two_k - 1) if a > 0 else two_k - 1
        tl = last[i]
        s = tl + k
        while (s + b) % two_k not in (0, k):
            s += 1
        if s <= t_end:
            continue  # erased at preserve point s
        vals[i] = (tl + b) % two_k
    return vals


def test_atv_hand_table_k2_g4():
    rows = read_golden("atv_k2_g4_hand.txt")
    o = O.Oracle(k=2, g=4, **TINY)
    assert o.blocks() == (1, 1)
    for t_s, c0, pre, touched, post, active, w in rows:
        t = int(t_s)
        assert o.t == t and o.C0 == int(c0)
        assert o.pool()[0, 0, 0].tolist() == [int(v) for v in pre.split(",")]
        if touched != "-":
            for i in touched.split(","):
                o.touch(0, 0, 0, int(i))
        assert o.pool()[0, 0, 0].tolist() == [int(v) for v in post.split(",")]
        assert o.detect() == 0
        W, _, _ = o.weights()
        assert W[0, 0, 0] == int(w) == active.count("1")
        o.advance()


@pytest.mark.parametrize("g,k", [(16, 3), (7, 3), (128, 4), (256, 10), (512, 60), (128, 1),
                                 (40, 300)])
def test_atv_equals_exact_last_set(g, k):
    """S:74 / P:241: for random touch schedules, the weight equals the number of ATs
    set within the latest k' slices (current slice included), for k' in {1, k/2, k};
    the stored values equal the exact model above both before and after preserve."""
    rng = np.random.default_rng(1000 * g + k)
    n_slices = 3 * k + 12 if k < 100 else 2 * k + 40
    for kp in sorted({1, max(1, k // 2), k}):
        o = O.Oracle(k=k, g=g, k_prime=kp, **MICRO)
        last = np.full(g, -1, dtype=np.int64)
        for t in range(n_slices):
            dens = rng.choice([0.0, 0.02, 0.2, 0.7])
            touched = np.nonzero(rng.random(g) < dens)[0]
            for i in touched:
                o.touch(0, 0, 0, int(i))
            last[touched] = t
            # values during slice t (preserve for t applied, touches of t applied)
            exp = _expected_after(last, t, k, g)
            assert (o.pool()[0, 0, 0].astype(np.int64) == exp).all(), (t, kp)
            assert o.detect() == 0
            W, _, _ = o.weights()
            truth = int(((last >= 0) & (t - last <= kp - 1)).sum())
            assert W[0, 0, 0] == truth, (t, kp)
            o.advance()
            exp = _expected_after(last, t + 1, k, g)
            assert (o.pool()[0, 0, 0].astype(np.int64) == exp).all(), (t + 1, kp)


def test_full_decay_after_2k_idle_slices():
    """after 2k slices without SetAT every AT is back to 2k."""
    k, g = 5, 40
    o = O.Oracle(k=k, g=g, **MICRO)
    for i in range(g):
        o.touch(0, 0, 0, i)
    for _ in range(2 * k):
        o.advance()
    assert (o.pool() == 2 * k).all()


def test_block_layout_paper_statement():
    """first 2k-1 blocks hold a ATs, the last b, a(2k-1)+b = g; block i has
    ACT (C0+i) mod 2k. Example S:119: g=1200, k=300, C0=7, AT 3 -> block 1 -> 8."""
    for g, k in [(128, 4), (256, 10), (512, 60), (512, 300), (4096, 300), (1200, 300), (7, 3)]:
        o = O.Oracle(k=k, g=g, **MICRO)
        a, b = o.blocks()
        assert a * (2 * k - 1) + b == g and b >= a >= 0
        sizes = np.bincount([o.block(i) for i in range(g)], minlength=2 * k)
        if a > 0:
            assert (sizes[:2 * k - 1] == a).all() and sizes[2 * k - 1] == b
        else:
            assert sizes[2 * k - 1] == g
    o = O.Oracle(k=300, g=1200, **MICRO)
    for _ in range(7):
        o.advance()
    assert o.C0 == 7 and o.block(3) == 1 and o.act(3) == 8
    o.touch(0, 0, 0, 3)
    assert o.pool()[0, 0, 0, 3] == 8


def test_preserve_touches_only_two_blocks_per_slice():
    """P:256 'only AT in two blocks need to apply preserveAT': count ATs whose
    value changes through advance() on a pool fully set to values that any
    preserve point would erase; it equals the sizes of the blocks whose new ACT
    is 0 or k (closed form)."""
    k, g = 6, 60
    o = O.Oracle(k=k, g=g, **MICRO)
    a, b = o.blocks()
    for t in range(3 * k):
        # set every AT of ATV(0,0,0) to a value that is erasable by either rule:
        # value 0 is erased by both the act==0 and the act==k rule
        pool = o.pool()
        pool[0, 0, 0, :] = 0
        o.set_pool(pool)
        o.advance()
        after = o.pool()[0, 0, 0]
        changed = int((after != 0).sum())
        acts = [(o.C0 + bl) % (2 * k) for bl in range(2 * k)]
        sizes = [a] * (2 * k - 1) + [b]
        expect = sum(sz for bl, sz in enumerate(sizes) if acts[bl] % k == 0)
        assert changed == expect
