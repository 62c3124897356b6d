"""GPU parity: the sm_100a path through the C-ABI against the CPU oracle, slice by
slice, on the seeded BASELINE.json traces and on edge cases.
Pool and CSIP bit-exact, NAT exact, estimates within 1e-6 relative (tests/parity.py)."""
import numpy as np
import pytest
import torch

from gen import PRESETS, Generator
from oracle import oracle as O
from paper_1807_01527_b200 import asse
from parity import compare_pool, compare_reports, step_both, to_device

pytestmark = pytest.mark.gpu


def _pair(name, **over):
    p = dict(PRESETS[name], **over)
    return asse.Asse(**p), O.Oracle(**p), p


def test_keys_and_initial_pool(cuda_device):
    dev, ora, p = _pair("C1")
    assert dev.keys() == ora.keys()          # both derived from the seed independently (A14)
    compare_pool(dev.pool(), ora.pool(), "init")
    assert dev.stats()["code_bytes"] == 1
    assert dev.stats()["w_theta"] == int(np.ceil(O.w_theta(p["g"], p["theta"])))


def test_c1_all_slices(cuda_device):
    dev, ora, p = _pair("C1")
    g = Generator("C1")
    for t in range(p["T"]):
        rep_d, rep_o = step_both(dev, ora, g.slice(t), p["theta"], "C1 t=%d" % t)
        assert len(rep_o) > 0 or t == 0
        # mode 0 (est >= theta) re-read from the same closed slice
        above = dev.fetch_reports(0)
        exp = rep_o[(rep_o["flags"] & 2) != 0]
        compare_reports(above, exp, p["theta"], "C1 mode0 t=%d" % t)


def test_c2_all_slices(cuda_device):
    dev, ora, p = _pair("C2")
    g = Generator("C2")
    for t in range(p["T"]):
        step_both(dev, ora, g.slice(t), p["theta"], "C2 t=%d" % t, check_pool=(t % 3 == 0 or t > 26))


@pytest.mark.parametrize("name,N,T", [("C3", 1_000_000, 5), ("C4", 600_000, 4)])
def test_backbone_geometries_reduced_n(cuda_device, name, N, T):
    """C3 (u8 codes, k=60) and C4 (u16 codes, k=300, g < 2k so a = 0, A7) geometry."""
    dev, ora, p = _pair(name)
    g = Generator(name, N=N)
    for t in range(T):
        step_both(dev, ora, g.slice(t), p["theta"], "%s t=%d" % (name, t))
    if name == "C4":
        assert dev.stats()["code_bytes"] == 2


@pytest.mark.parametrize("name,T", [("C3", 2), ("C4", 2)])
def test_full_size_slices(cuda_device, name, T):
    """BASELINE.json full per-slice sizes (20M / 10M packets), the launch configuration
    bench.py times; full pool and CSIP compared for the first slices (C5 at 100M packets:
    tests/test_gpu_window.py::test_full_size_c5_pipelined)."""
    dev, ora, p = _pair(name)
    g = Generator(name)
    for t in range(T):
        step_both(dev, ora, g.slice(t, threads=16), p["theta"], "%s full t=%d" % (name, t))


def test_gpu_generator_matches_host(cuda_device):
    for name in ("C1", "C2", "C3", "C4"):
        g = Generator(name)
        n = min(300_000, (g.N - 7) // 3)
        out = torch.empty(2 * n, dtype=torch.int32, device="cuda")
        g.slice_cuda(2, out.data_ptr(), j0=7, n=n, stride=3)
        torch.cuda.synchronize()
        host = g.slice(2, j0=7, n=n, stride=3)
        assert (out.cpu().numpy().view(np.uint32).reshape(-1, 2) == host).all(), name


def test_long_run_sweeps_small_geometry(cuda_device):
    """k = 300 with g = 128 < 2k (every AT in block 2k-1, swept every k slices,
    A7): 700 slices cross both sweep points twice; pool parity after every slice."""
    geo = dict(k=300, r=4, c=8, u=4, s=7, g=128, theta=200.0, seed=42)
    dev, ora = asse.Asse(**geo), O.Oracle(**geo)
    rng = np.random.default_rng(3)
    hosts = rng.integers(0, 2 ** 32, 64).astype(np.uint32)
    for t in range(700):
        n = int(rng.integers(0, 3000))
        pk = np.stack([hosts[rng.integers(0, 64, n)],
                       rng.integers(0, 2 ** 32, n).astype(np.uint32)], 1).astype(np.uint32)
        step_both(dev, ora, pk, geo["theta"], "long t=%d" % t, check_pool=(t % 7 == 0 or t in (299, 300, 301, 599, 600, 601)))


@pytest.mark.parametrize("k,kp", [(1, 1), (4, 2), (10, 1), (60, 17), (100, 100), (600, 300)])
def test_window_variants(cuda_device, k, kp):
    """discrete window k = 1, k' < k (Alg. 1), and u16 codes at k = 100."""
    geo = dict(k=k, k_prime=kp, r=4, c=10, u=4, s=6, g=256, theta=300.0, seed=9)
    dev, ora = asse.Asse(**geo), O.Oracle(**geo)
    g = Generator("C2", N=150_000)
    for t in range(min(2 * k + 3, 14)):
        step_both(dev, ora, g.slice(t), geo["theta"], "k=%d k'=%d t=%d" % (k, kp, t))


@pytest.mark.parametrize("g,k", [(1024, 10), (2048, 60), (4096, 300), (4096, 4)])
def test_large_atv(cuda_device, g, k):
    """g > 512 (the paper's own g = 4096): an ATV spans g/512 fold chunks."""
    geo = dict(k=k, r=4, c=8, u=4, s=7, g=g, theta=1024.0, seed=31)
    dev, ora = asse.Asse(**geo), O.Oracle(**geo)
    gen = Generator("C2", N=300_000)
    for t in range(5):
        step_both(dev, ora, gen.slice(t), geo["theta"], "g=%d k=%d t=%d" % (g, k, t))


@pytest.mark.parametrize("name,N", [("C1", None), ("C3", 1_000_000)])
def test_mod_p_mangling(cuda_device, name, N):
    """the paper-literal mod-p mangling (config mangle = 1)."""
    dev, ora, p = _pair(name, mangle=1)
    assert dev.keys() == ora.keys()
    g = Generator(name, N=N)
    for t in range(4):
        step_both(dev, ora, g.slice(t), p["theta"], "%s mod-p t=%d" % (name, t))
    # hosts whose image A x mod p lands in [2^32, p) take the cycle walk on both sides
    A, Ai, _ = ora.keys()
    P = 2 ** 32 + 15
    walkers = [x for x in ((Ai * t) % P for t in range(2 ** 32, P)) if x < 2 ** 32]
    assert walkers
    rng = np.random.default_rng(1)
    rows = [np.stack([np.full(3000, x, np.uint64), rng.integers(0, 2 ** 32, 3000)], 1) for x in walkers]
    pk = np.concatenate([g.slice(5, n=100_000).astype(np.uint64)] + rows).astype(np.uint32)
    rd, ro = step_both(dev, ora, pk, p["theta"], "%s mod-p walkers" % name)
    assert set(walkers) <= set(ro["ip"].tolist())


def test_edge_cases_empty_ragged_misaligned_split(cuda_device):
    dev, ora, p = _pair("C1")
    g = Generator("C1")
    # empty slice
    step_both(dev, ora, np.zeros((0, 2), np.uint32), p["theta"], "empty")
    # one packet, then odd counts, a misaligned buffer and several scan calls per slice
    step_both(dev, ora, g.slice(0, n=1), p["theta"], "n=1")
    step_both(dev, ora, g.slice(1, n=12345), p["theta"], "odd", offset=1)
    step_both(dev, ora, g.slice(2), p["theta"], "split", split=7)
    step_both(dev, ora, g.slice(3, n=99999), p["theta"], "split+misaligned", split=3, offset=1)


def test_order_invariance_and_host_ingest(cuda_device):
    """concurrent SetATs are order independent; the host-buffer entry point
    (double-buffered H2D) gives the identical state."""
    p = dict(PRESETS["C2"])
    a, b, c = asse.Asse(**p), asse.Asse(**p), asse.Asse(**p)
    g = Generator("C2")
    rng = np.random.default_rng(0)
    for t in range(3):
        pk = g.slice(t)
        d1, _ = to_device(pk)
        d2, _ = to_device(pk[rng.permutation(len(pk))])
        a.scan_slice(d1)
        b.scan_slice(d2)
        c.scan_slice_host(np.ascontiguousarray(pk))
        ra, rb, rc = a.end_slice(), b.end_slice(), c.end_slice()
        assert (ra == rb).all() and (ra == rc).all()
        pa = a.pool()
        assert (pa == b.pool()).all() and (pa == c.pool()).all()


def test_overflow_reported_and_state_continues(cuda_device):
    geo = dict(PRESETS["C1"], max_candidates=50)
    dev, ora = asse.Asse(**geo), O.Oracle(**geo)
    g = Generator("C1")
    for t in range(4):
        pk = g.slice(t)
        d, ptr = to_device(pk)
        dev.scan_slice(ptr, len(pk))
        ora.scan(pk)
        st_o = ora.detect()
        ora.advance()
        try:
            dev.end_slice()
            st_d = 0
        except asse.AsseError as e:
            st_d = e.status
        assert (st_d == asse.E_OVERFLOW) == (st_o == -4), t
        compare_pool(dev.pool(), ora.pool(), "overflow t=%d" % t)


def test_state_machine_errors(cuda_device):
    geo = dict(PRESETS["C1"], n_slices=2)
    dev = asse.Asse(**geo)
    dev.end_slice()
    dev.end_slice()
    with pytest.raises(asse.AsseError) as e:
        dev.end_slice()
    assert e.value.status == asse.E_STATE
    with pytest.raises(asse.AsseError):
        asse.Asse(**dict(PRESETS["C1"], g=100))



@pytest.mark.parametrize("k,T", [(63, 2 * 63 + 3), (64, 2 * 64 + 3), (16383, 6)])
def test_code_width_boundaries_and_max_k(cuda_device, k, T):
    """Code-width edges (A2): k = 63 is the largest window with 8-bit codes (2k = 126, the
    EMPTY value 2k still below the guard bit), k = 64 the first with 16-bit codes; both run
    past their erasures (t >= k) and the C0 wrap (t = 2k). k = 16383 is validate()'s maximum
    (15-bit device codes): with g = 256 < 2k every AT sits in block 2k-1 (A7), so the block
    ACT starts at 2k-1 = 32765 and the checkAT intervals wrap from the first slice."""
    geo = dict(k=k, r=4, c=8, u=4, s=7, g=256, theta=300.0, seed=41)
    dev, ora = asse.Asse(**geo), O.Oracle(**geo)
    assert dev.stats()["code_bytes"] == (1 if 2 * k <= 126 else 2)
    gen = Generator("C2", N=30_000)
    for t in range(T):
        step_both(dev, ora, gen.slice(t), geo["theta"], "k=%d t=%d" % (k, t))
    assert dev.clock() == (T, T % (2 * k))


@pytest.mark.parametrize("r,c,u,s", [(2, 15, 4, 13), (3, 12, 4, 8), (5, 9, 2, 6), (8, 8, 4, 3), (4, 12, 0, 7),
                                     (4, 6, 12, 5)])
def test_row_counts_and_frame_extremes(cuda_device, r, c, u, s):
    """Geometries off the BASELINE shape (validate()'s range): r = 2, 3, 5 and 8
    rows (the scan falls back to k_scan, which handles any r; the fold and the join are
    generic in r), a single frame (u = 0, 32-bit LBS) and 4096 frames of 64 estimators
    (u = 12). C1's planted super points make CSIP non-empty; pool, CSIP, NAT and the
    estimates equal the oracle after every slice past the first erasures (k = 4)."""
    geo = dict(k=4, r=r, c=c, u=u, s=s, g=256, theta=1024.0, seed=43)
    dev, ora = asse.Asse(**geo), O.Oracle(**geo)
    gen = Generator("C1")
    seen = 0
    for t in range(10):
        rep_d, _ = step_both(dev, ora, gen.slice(t), geo["theta"], "r=%d c=%d u=%d t=%d" % (r, c, u, t))
        seen += len(rep_d)
    assert seen > 0                                   # the join produced candidates
    assert dev.stats()["scan_own_launches"] == 0 or r == 4
