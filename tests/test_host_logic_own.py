"""Host-side arithmetic of the packet-owned scan (asse_api.cu, asse_scan_own.cuh), checked on
CPU: the owner choice (frame x word group of BH(bip)), the slice layout and its write-back
mapping must partition the touch bitmap exactly; the 8-byte entry must carry everything the
owner needs to reproduce k_scan's SetAT targets (Alg. 3; frames P:297; column
windows P:314-324); the queue rings and shared memory must hold a round's worst case."""
import numpy as np
import pytest

from gen import PRESETS

KOWN_CAP, KBIN_QG, KOWN_QCAP, KOWN_MAX_OWNERS, KOWN_RING = 30, 6, 1024, 128, 2   # asse_scan_own.cuh
OPTIN = 232448                                                                     # B200 opt-in smem / block


def own_geometry(p, sms):
    """Mirror of asse_init's packet-owned-scan setup."""
    F, wpa = 1 << p["u"], p["g"] // 32
    lg_wpa = 0
    while (1 << lg_wpa) < wpa:
        lg_wpa += 1
    lg_ngrp = 0
    while lg_ngrp < lg_wpa and (F << (lg_ngrp + 1)) <= sms:
        lg_ngrp += 1
    lg_wg = lg_wpa - lg_ngrp
    O = F << lg_ngrp
    tile = min(2048, max(1024, O * 16) // 1024 * 1024) * 8
    slice_words = p["r"] << (p["c"] + lg_wg)
    smem = KOWN_RING * tile + 2 * O * KOWN_CAP * 8 + 2 * ((O * 4 + 15) & ~15) + 16 + slice_words * 4
    ok = (p["r"] == 4 and (1 << lg_wpa) == wpa and O <= sms and lg_wg <= p["u"] and O <= KOWN_MAX_OWNERS
          and O >= 2 and -(-sms // KBIN_QG) * KOWN_CAP <= KOWN_QCAP and slice_words <= (1 << 20)
          and smem + 1024 <= OPTIN)
    return dict(F=F, wpa=wpa, lg_ngrp=lg_ngrp, lg_wg=lg_wg, O=O, tile=tile, slice_words=slice_words,
                smem=smem, ok=ok)


@pytest.mark.parametrize("sms", [132, 148, 160])
def test_geometry_admission(sms):
    for name in ("C1", "C2", "C3", "C4", "C5"):
        g = own_geometry(PRESETS[name], sms)
        assert g["ok"], (name, g)
    g = own_geometry(PRESETS["C3"], sms)
    assert (g["O"], g["lg_wg"], g["slice_words"]) == (128, 1, 32768)   # 128 owners x 128 KiB
    assert not own_geometry(PRESETS["PAPER"], sms)["ok"]                # 4 MiB slices


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_slices_partition_the_bitmap(name):
    """(owner, slice word) <-> global touch word is a bijection, and the kernel's write-back
    formula maps each slice word back to the word it stands for."""
    p = PRESETS[name]
    g = own_geometry(p, 148)
    F, c, wpa, lg_wg = g["F"], p["c"], g["wpa"], g["lg_wg"]
    E = 1 << c
    y, z, x, w = np.meshgrid(np.arange(p["r"]), np.arange(F), np.arange(E), np.arange(wpa), indexing="ij")
    y, z, x, w = (a.ravel().astype(np.int64) for a in (y, z, x, w))
    gword = (((y * F + z) << c) + x) * wpa + w                 # k_scan's target word
    owner = (z << g["lg_ngrp"]) | (w >> lg_wg)
    sw = (((y << c) | x) << lg_wg) | (w & ((1 << lg_wg) - 1))
    assert owner.max() < g["O"] and sw.max() < g["slice_words"]
    key = owner * g["slice_words"] + sw
    assert len(np.unique(key)) == len(key) == g["O"] * g["slice_words"]
    # write-back (asse_scan_own.cuh, end of k_scan_own): z = o >> lg_ngrp, grp = o & (NGRP-1)
    zz, grp = owner >> g["lg_ngrp"], owner & ((1 << g["lg_ngrp"]) - 1)
    yx, sub = sw >> lg_wg, sw & ((1 << lg_wg) - 1)
    yy, xx = yx >> c, yx & (E - 1)
    back = (yy * (F << c) + xx) * wpa + (zz << c) * wpa + grp * (1 << lg_wg) + sub
    assert (back == gword).all()


def touch_bit_u8(i):
    return ((i >> 4) & 1) * 16 + 4 * (i & 3) + ((i >> 2) & 3)


def test_entry_reproduces_scan_targets():
    """Producer: owner = (f & fmask) << lg_ngrp | i >> (5 + lg_wg); entry = (f & ~fmask) |
    ((i >> 5) & wgm), touch mask of i. Owner: L = e >> u, sub = e & fmask, r windows of L.
    The r (word, bit) pairs it sets are exactly k_scan's for the same (f(aip), i)."""
    p = PRESETS["C3"]
    g = own_geometry(p, 148)
    u, c, F, wpa, lg_wg = p["u"], p["c"], g["F"], g["wpa"], g["lg_wg"]
    W, fm, cm = 32 - u, (1 << u) - 1, (1 << c) - 1
    shift = [(p["s"] * yy) % W for yy in range(p["r"])]
    rng = np.random.default_rng(5)
    h = rng.integers(0, 2 ** 32, 20000, dtype=np.uint64)
    i = rng.integers(0, p["g"], 20000, dtype=np.uint64)
    # k_scan (scan_pair): z, LBS, wrap-around windows, ATV, word, bit
    z = h & np.uint64(fm)
    L = h >> np.uint64(u)
    D = L | (L << np.uint64(W))
    ref = []
    for yy in range(p["r"]):
        x = (D >> np.uint64(shift[yy])) & np.uint64(cm)
        atv = (np.uint64(yy) << np.uint64(u + c)) + (z << np.uint64(c)) + x
        ref.append(atv * np.uint64(wpa) + (i >> np.uint64(5)))
    # producer entry, owner decode, slice word -> global word (write-back)
    owner = (z << np.uint64(g["lg_ngrp"])) | (i >> np.uint64(5 + lg_wg))
    e = (h & np.uint64(0xFFFFFFFF ^ fm)) | ((i >> np.uint64(5)) & np.uint64((1 << lg_wg) - 1))
    Lo = e >> np.uint64(u)
    sub = e & np.uint64(fm)
    Do = Lo | (Lo << np.uint64(W))
    zz, grp = owner >> np.uint64(g["lg_ngrp"]), owner & np.uint64((1 << g["lg_ngrp"]) - 1)
    for yy in range(p["r"]):
        x = (Do >> np.uint64(shift[yy])) & np.uint64(cm)
        sw = (((np.uint64(yy) << np.uint64(c)) | x) << np.uint64(lg_wg)) | sub
        yx, sb = sw >> np.uint64(lg_wg), sw & np.uint64((1 << lg_wg) - 1)
        gw = ((yx >> np.uint64(c)) * np.uint64(F << c) + (yx & np.uint64(cm))) * np.uint64(wpa) + \
            (zz << np.uint64(c)) * np.uint64(wpa) + grp * np.uint64(1 << lg_wg) + sb
        assert (gw == ref[yy]).all()
    assert (owner < g["O"]).all()
    # the touch mask depends on i mod 32 only, through a permutation of the word's bits
    assert sorted(touch_bit_u8(v) for v in range(32)) == list(range(32))
    assert all(touch_bit_u8(v) == touch_bit_u8(v + 32 * k) for v in range(32) for k in range(16))


@pytest.mark.parametrize("sms", [132, 148, 160])
def test_queue_ring_holds_a_round(sms):
    """Every producer of a group filling its owner's bin in one round fits the ring, and
    the padded (even) bins keep every copy 16-B aligned."""
    per_group = -(-sms // KBIN_QG)
    assert per_group * KOWN_CAP <= KOWN_QCAP
    assert KOWN_CAP % 2 == 0 and (KOWN_CAP * 8) % 16 == 0 and KOWN_QCAP & (KOWN_QCAP - 1) == 0
