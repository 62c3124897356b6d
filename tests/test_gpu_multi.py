"""Multi-GPU merge path on ONE GPU: D 'virtual ranks' (contexts with world = D) scan
round-robin shards into their own touch bitmaps; the same k_merge_or kernel the
real NVLink path runs ORs them (A26) with the caller ordering the phases
(asse_attach_peers sync_mode 1 — no kernel waits on another). Every rank must end
with the pool and reports of a single context fed the whole slice, and of the
oracle. The device-barrier variant (sync_mode 0) needs one process per GPU."""
import numpy as np
import pytest
import torch

from gen import PRESETS, Generator
from oracle import oracle as O
from paper_1807_01527_b200 import asse
from paper_1807_01527_b200.dist import attach_local_peers, shard_slots
from parity import compare_pool, compare_reports, to_device

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shard", [0, 1])
@pytest.mark.parametrize("name,D,N,T", [("C1", 2, None, 5), ("C2", 4, 600_000, 4),
                                        ("C3", 8, 2_000_000, 3), ("C4", 16, 400_000, 3)])
def test_virtual_ranks_merge_equals_single(cuda_device, name, D, N, T, shard):
    """shard 0: replicated pools (option R); shard 1: rank d keeps frames
    [d F/D, (d+1) F/D) (option S) and the reports are gathered from every rank."""
    _run_virtual_ranks(name, D, N, T, shard, 0)


@pytest.mark.parametrize("shard", [0, 1])
@pytest.mark.parametrize("name,D,N,T", [("C3", 2, 3_000_000, 2), ("C4", 4, 2_400_000, 2)])
def test_virtual_ranks_binned_scan(cuda_device, name, D, N, T, shard):
    """The same with every rank's scan forced onto k_scan_bin (its write-back lands in the
    rank's peer-visible touch bitmap)."""
    _run_virtual_ranks(name, D, N, T, shard, 2)


@pytest.mark.parametrize("shard", [0, 1])
@pytest.mark.parametrize("name,D,N,T", [("C3", 2, 3_000_000, 2), ("C4", 8, 4_000_000, 2)])
def test_virtual_ranks_packet_owned_scan(cuda_device, name, D, N, T, shard):
    """The same with every rank's scan forced onto k_scan_own (the default scan at C3-C5;
    its write-back lands in the rank's peer-visible touch bitmap)."""
    _run_virtual_ranks(name, D, N, T, shard, 3)


def _run_virtual_ranks(name, D, N, T, shard, variant):
    p = dict(PRESETS[name])
    ranks = [asse.Asse(**dict(p, world=D, rank=d, frame_shard=shard)) for d in range(D)]
    for ctx in ranks:
        ctx.set_scan_variant(variant)
    bufs = attach_local_peers(ranks)
    single = asse.Asse(**p)
    ora = O.Oracle(**p)
    g = Generator(name, N=N)
    for t in range(T):
        pk = g.slice(t)
        keep = []
        for d, ctx in enumerate(ranks):
            j0, stride, n = shard_slots(len(pk), d, D)
            dpk, ptr = to_device(np.ascontiguousarray(pk[j0::stride]))
            keep.append(dpk)
            ctx.scan_slice(ptr, n)
        torch.cuda.synchronize()
        for ctx in ranks:
            ctx.merge()
        torch.cuda.synchronize()
        if shard:
            for ctx in ranks:
                ctx.end_slice_begin()
            torch.cuda.synchronize()
        reps = [ctx.end_slice(1) for ctx in ranks]
        dfull, ptr = to_device(pk)
        single.scan_slice(ptr, len(pk))
        rs = single.end_slice(1)
        ora.scan(pk)
        ro = ora.end_slice(1)
        compare_reports(rs, ro, p["theta"], "%s single t=%d" % (name, t))
        if shard:   # the rank pools are the frame slices of the whole pool
            pool0 = np.concatenate([ctx.pool() for ctx in ranks], axis=1)
        else:
            pool0 = ranks[0].pool()
        compare_pool(pool0, ora.pool(), "%s merged t=%d" % (name, t))
        for d in range(D):
            compare_reports(reps[d], ro, p["theta"], "%s rank %d t=%d" % (name, d, t))
            if d and not shard:
                assert (ranks[d].pool() == pool0).all()
    del bufs


@pytest.mark.slow
@pytest.mark.parametrize("D,shard", [(8, 1), (2, 0)])
def test_virtual_ranks_full_size_c5(cuda_device, D, shard):
    """BASELINE.json configs[4] at full size: the 100M-packet C5 slice split round-robin
    over D ranks (12.5M / 50M packets each, the packet-owned scan on every rank), merged
    and closed; every rank equals the oracle fed the whole slice ("results must be
    identical for every D")."""
    _run_virtual_ranks("C5", D, None, 2, shard, 0)
