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
