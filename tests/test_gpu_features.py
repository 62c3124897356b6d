"""SURVEY §8(f) rows built on the same kernels: window queries k' < k, checkpoint /
restore, and the discrete-window mode with the paper's boundary-spanning example."""
import numpy as np
import pytest
import torch

from gen import PRESETS, Generator
from oracle import oracle as O
from paper_1807_01527_b200 import asse
from parity import compare_pool, compare_reports, to_device

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,N", [("C2", 400_000), ("C3", 1_000_000)])
def test_query_window_equals_oracle_with_that_kprime(cuda_device, name, N):
    """asse_query_window(k') after closing slice t == the oracle run with k'."""
    p = dict(PRESETS[name])
    k = p["k"]
    kps = [1, k // 2, k - 1]
    dev = asse.Asse(**p)
    oras = {kp: O.Oracle(**dict(p, k_prime=kp)) for kp in kps}
    g = Generator(name, N=N)
    for t in range(min(k + 2, 10)):
        pk = g.slice(t)
        d, ptr = to_device(pk)
        dev.scan_slice(ptr, len(pk))
        dev.end_slice(1)
        for kp in kps:
            oras[kp].scan(pk)
            ro = oras[kp].end_slice(1)
            rd = dev.query_window(kp, 1)
            compare_reports(rd, ro, p["theta"], "%s t=%d k'=%d" % (name, t, kp))
    with pytest.raises(asse.AsseError):
        dev.query_window(k)
    # the pool is untouched by queries
    compare_pool(dev.pool(), oras[kps[-1]].pool(), "pool after queries")


@pytest.mark.parametrize("name", ["C1", "C4"])
def test_checkpoint_roundtrip(cuda_device, tmp_path, name):
    """u8 (C1) and u16 (C4, k = 300) pools: a resumed run equals the uninterrupted one."""
    p = dict(PRESETS[name], N=200_000) if name == "C4" else dict(PRESETS[name])
    a = asse.Asse(**p)
    g = Generator(name, N=p["N"])
    for t in range(3):
        d, ptr = to_device(g.slice(t))
        a.scan_slice(ptr, g.N)
        a.end_slice()
    path = str(tmp_path / "c1.ckpt")
    a.save_state(path)
    b = asse.Asse(**p)
    b.load_state(path)
    assert b.clock() == a.clock()
    assert (b.pool() == a.pool()).all()
    for t in range(3, 6):
        d, ptr = to_device(g.slice(t))
        a.scan_slice(ptr, g.N)
        b.scan_slice(ptr, g.N)
        ra, rb = a.end_slice(), b.end_slice()
        assert len(ra) == len(rb) and (ra == rb).all()
    assert (a.pool() == b.pool()).all()
    other = asse.Asse(**dict(p, seed=99))
    with pytest.raises(asse.AsseError):
        other.load_state(path)


def test_boundary_spanner_sliding_vs_discrete(cuda_device):
    """a host with 512 peers before and 512 after a window boundary is missed
    by discrete windows and found by the sliding window spanning the boundary
    (scaled: 200 + 200 peers, theta = 300, g = 512)."""
    geo = dict(r=4, c=10, u=4, s=6, g=512, theta=300.0, seed=13)
    H = 0x0A000001
    rng = np.random.default_rng(4)

    def slice_pk(t):
        bg = np.stack([rng.integers(0, 2 ** 32, 5000), rng.integers(0, 2 ** 32, 5000)], 1)
        if t in (1, 2):
            bips = np.arange(200, dtype=np.uint64) + 1000 * t
            bg = np.concatenate([bg, np.stack([np.full(200, H), bips], 1)])
        return np.ascontiguousarray(bg.astype(np.uint32))

    slices = [slice_pk(t) for t in range(4)]
    # sliding window of k = 2 slices, one slice = one time unit
    sl = asse.Asse(k=2, **geo)
    found = []
    for t, pk in enumerate(slices):
        d, ptr = to_device(pk)
        sl.scan_slice(ptr, len(pk))
        found.append(H in set(sl.end_slice(0)["ip"].tolist()))
    assert found == [False, False, True, False]
    # discrete windows of the same length (k = 1, one slice = two time units)
    ds = asse.Asse(k=1, **geo)
    for a, b in ((0, 1), (2, 3)):
        for pk in (slices[a], slices[b]):
            d, ptr = to_device(pk)
            ds.scan_slice(ptr, len(pk))
        assert H not in set(ds.end_slice(0)["ip"].tolist())


@pytest.mark.parametrize("name,N,T,variant", [("C1", 200_000, 6, 0), ("C3", 1_500_000, 4, 2)])
def test_async_end_slice_pipeline(cuda_device, name, N, T, variant):
    """asse_end_slice_async + asse_end_slice_wait with the next slice's scan issued in
    between (the bench's pipelined step) gives every slice's reports and the final pool
    of the oracle run; other calls are refused while results are pending."""
    p = dict(PRESETS[name])
    dev, ora = asse.Asse(**p), O.Oracle(**p)
    dev.set_scan_variant(variant)
    g = Generator(name, N=N)
    live, expect = [], None
    for t in range(T):
        pk = g.slice(t)
        d, ptr = to_device(pk)
        live = (live + [d])[-2:]                 # device input must outlive its scan
        dev.scan_slice(ptr, len(pk))
        ora.scan(pk)
        if t:
            compare_reports(dev.end_slice_wait(), expect, p["theta"], "%s async t=%d" % (name, t - 1))
        dev.end_slice_async(1)
        expect = ora.end_slice(1)
        if t == 1:
            with pytest.raises(asse.AsseError):
                dev.pool()
            with pytest.raises(asse.AsseError):
                dev.end_slice_async(1)
    compare_reports(dev.end_slice_wait(), expect, p["theta"], "%s async last" % name)
    with pytest.raises(asse.AsseError):
        dev.end_slice_wait()
    compare_pool(dev.pool(), ora.pool(), "%s async pool" % name)
    assert dev.clock()[0] == T


def test_checkpoint_rejects_mangle_and_clock_mismatch(cuda_device, tmp_path):
    """Version-3 header: a pool saved with mangle = 0 is refused by a mangle = 1 context
    (A8: the key A and the host -> ATV map differ), and a header whose C0 is not
    t mod 2k is refused."""
    import struct
    p = dict(PRESETS["C1"])
    a = asse.Asse(**p)
    g = Generator("C1")
    for t in range(2):
        d, ptr = to_device(g.slice(t))
        a.scan_slice(ptr, g.N)
        a.end_slice()
    path = str(tmp_path / "c1.ckpt")
    a.save_state(path)
    with pytest.raises(asse.AsseError) as e:
        asse.Asse(**dict(p, mangle=1)).load_state(path)
    assert e.value.status == asse.E_PARAM and "mangl" in str(e.value)
    raw = bytearray(open(path, "rb").read())
    assert raw[:8] == b"ASSECKPT" and struct.unpack_from("<I", raw, 8)[0] == 3
    # header: magic 8 | version, code_bytes | k, kp, r, c, u, s, g | world, rank, shard |
    # mangle, pad | theta | seed | t | C0
    off_c0 = 8 + 4 * 2 + 4 * 7 + 4 * 3 + 4 * 2 + 8 + 8 + 8
    assert struct.unpack_from("<I", raw, off_c0)[0] == a.clock()[1] == 2
    struct.pack_into("<I", raw, off_c0, 3)
    bad = str(tmp_path / "bad.ckpt")
    open(bad, "wb").write(bytes(raw))
    with pytest.raises(asse.AsseError) as e:
        asse.Asse(**p).load_state(bad)
    assert e.value.status == asse.E_PARAM


@pytest.mark.parametrize("variant", [1, 3])
def test_side_stream_scan_after_async_end_slice(cuda_device, variant):
    """A scan issued on a caller stream right after asse_end_slice_async must run after
    that slice's fold (which reads and clears the touch bitmap): slice by slice equal to
    the oracle (the caller stream now waits for the context stream)."""
    p = dict(PRESETS["C3"])
    dev, ora = asse.Asse(**p), O.Oracle(**p)
    dev.set_scan_variant(variant)
    side = torch.cuda.Stream()
    g = Generator("C3", N=3_000_000)
    live, expect = [], None
    for t in range(4):
        pk = g.slice(t)
        d, ptr = to_device(pk)
        live = (live + [d])[-2:]
        dev.scan_slice(ptr, len(pk), stream=side.cuda_stream)
        ora.scan(pk)
        if t:
            compare_reports(dev.end_slice_wait(), expect, p["theta"], "side t=%d" % (t - 1))
        dev.end_slice_async(1)
        expect = ora.end_slice(1)
    compare_reports(dev.end_slice_wait(), expect, p["theta"], "side last")
    compare_pool(dev.pool(), ora.pool(), "side pool")
