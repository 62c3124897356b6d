"""Host-side arithmetic of the binned scan (asse_api.cu, asse_scan_bin.cuh), checked
exhaustively on CPU: the owner of a touch word is (w * ceil(2^40 / wpo)) >> 40, which must
equal w // wpo for every binned word of every geometry the library accepts, and the queue
rings must hold a round's worst case (every producer group member's bin full)."""
import numpy as np
import pytest

from gen import PRESETS

KBIN_CAP, KBIN_QG, KBIN_QCAP = 88, 4, 4096     # asse_scan_bin.cuh


def bin_geometry(p, sms, rr=1):
    F, E, wpa = 1 << p["u"], 1 << p["c"], p["g"] // 32
    row_words = F * E * wpa
    if (p["r"] * row_words) // sms <= 16384:
        rr = 0
    if ((p["r"] - rr) * row_words) // sms <= 256:
        rr = 0
    words = (p["r"] - rr) * row_words
    wpo = ((words + sms - 1) // sms + 3) & ~3
    inv = min(0xFFFFFFFF, ((1 << 40) + wpo - 1) // wpo)
    return words, wpo, inv, rr


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
@pytest.mark.parametrize("sms", [132, 148, 160])
def test_owner_formula_exact(name, sms):
    words, wpo, inv, rr = bin_geometry(PRESETS[name], sms)
    assert wpo > 256 and inv < 2 ** 32 and words < 2 ** 25
    w = np.arange(words, dtype=np.uint64)
    owner = (w * np.uint64(inv)) >> np.uint64(40)
    assert (owner == w // np.uint64(wpo)).all()
    local = w - owner * np.uint64(wpo)
    assert int(local.max()) < wpo < 2 ** 27          # entry = local << 5 | bit fits in 32 bits
    assert int(owner.max()) < sms


@pytest.mark.parametrize("sms", [132, 148, 160])
def test_queue_ring_holds_a_round(sms):
    group = (sms + KBIN_QG - 1) // KBIN_QG           # producers per (owner, group) ring
    assert group * KBIN_CAP <= KBIN_QCAP             # a round never laps the ring


def _freepos(c, s, u, r):
    """Mirror of asse_init's join plan: per row y the window positions j of x_y whose LBS bit
    (s*y + j) mod W is not fixed by rows < y."""
    W = 32 - u
    known = [False] * W
    out = []
    for y in range(r):
        fp = [j for j in range(c) if not known[(s * y + j) % W]]
        for j in range(c):
            known[(s * y + j) % W] = True
        out.append(fp)
    return out


def _two_runs(fp):
    """Mirror of asse_init: (ok, n1, sh1, sh2) with bits [0, n1) << sh1, the rest << sh2."""
    nf = len(fp)
    n1 = 0
    while n1 < nf and fp[n1] == fp[0] + n1:
        n1 += 1
    n2 = 0
    while n1 + n2 < nf and fp[n1 + n2] == fp[n1] + n2:
        n2 += 1
    return n1 + n2 == nf, n1, (fp[0] if nf else 0), (fp[n1] - n1 if n1 < nf else 0)


def _admissible(c, s, u, r):
    """Mirror of validate(): completeness and at least one duplicate position."""
    W = 32 - u
    if c + s * (r - 1) < W or c + u > 24 or s > c:
        return False
    cover = [0] * W
    for y in range(r):
        for j in range(c):
            cover[(s * y + j) % W] += 1
    return min(cover) > 0 and max(cover) > 1


def test_restore_free_positions_are_two_runs_for_every_geometry():
    """asse_init rejects a join plan whose free positions are not two ascending runs; that
    must never happen for an admissible geometry (a window is a cyclic interval of the LBS
    and the bits fixed by earlier rows a growing one)."""
    n = 0
    for u in range(0, 17):
        for c in range(2, 23):
            for s in range(1, c + 1):
                for r in range(2, 9):
                    if not _admissible(c, s, u, r):
                        continue
                    n += 1
                    for fp in _freepos(c, s, u, r):
                        assert _two_runs(fp)[0], (c, s, u, r, fp)
    assert n > 1000


@pytest.mark.parametrize("c,s,u,r", [(12, 6, 4, 4), (9, 7, 4, 4), (10, 5, 4, 4), (9, 6, 3, 4), (14, 5, 4, 4),
                                     (8, 8, 8, 4), (11, 3, 2, 8), (6, 4, 12, 4)])
def test_restore_deposit_runs_equal_the_bit_loop(c, s, u, r):
    """k_restore enumerates the completions of x_y by depositing the bits of sub into the free
    positions; the two-run form (shifts of two masked parts) must equal the per-bit loop for
    every sub < 2^nf."""
    if not _admissible(c, s, u, r):
        pytest.skip("rejected by validate")
    for y, fp in enumerate(_freepos(c, s, u, r)):
        ok, n1, sh1, sh2 = _two_runs(fp)
        assert ok, (y, fp)
        if len(fp) > 16:
            continue
        m1 = (1 << n1) - 1
        for sub in range(1 << len(fp)):
            loop = 0
            for b, pos in enumerate(fp):
                loop |= ((sub >> b) & 1) << pos
            assert ((sub & m1) << sh1) | ((sub & ~m1) << sh2) == loop
