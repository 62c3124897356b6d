"""Multi-process (gloo, world_size 2, CPU) test of the N>1 path logic: packets
sharded round-robin across ranks (BASELINE.json.configs[4]), one local AT pool
per rank, merged every slice with the most-recent-wins combine (A26; SURVEY
App. A.4) before detection. The merged state and reports must equal a single
pool fed the whole slice. The GPU path implements the same merge as an OR of
per-slice touch bitmaps, which this combine rule justifies."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from gen import PRESETS, Generator
        from oracle import oracle as O
        from paper_1807_01527_b200.dist import shard_slots

        p = dict(PRESETS["C1"])
        g = Generator("C1")
        local = O.Oracle(**p)
        single = O.Oracle(**p) if rank == 0 else None
        ok = True
        for t in range(6):
            j0, stride, n = shard_slots(g.N, rank, world)
            local.scan(g.slice(t, j0=j0, stride=stride, n=n))
            mine = torch.from_numpy(local.pool().astype(np.int32).ravel())
            parts = [torch.empty_like(mine) for _ in range(world)]
            dist.all_gather(parts, mine)
            pools = [x.numpy().astype(np.uint16) for x in parts]
            merged = local.combine_min_age(pools)
            local.set_pool(merged)
            assert local.detect() == 0
            rep = local.reports()
            local.advance()
            if rank == 0:
                single.scan(g.slice(t))
                assert single.detect() == 0
                srep = single.reports()
                ok &= bool((merged.reshape(-1) == single.pool().reshape(-1)).all())
                ok &= len(srep) == len(rep) and bool((srep == rep).all())
                single.advance()
                ok &= bool((single.pool() == local.pool()).all())
        # every rank holds the same merged pool
        mine = torch.from_numpy(local.pool().astype(np.int32).ravel())
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine)
        ok &= all(bool((parts[0] == x).all()) for x in parts)
        q.put((rank, ok))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


def test_gloo_world2_sharded_pools_merge_to_single():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res


@pytest.mark.parametrize("n,world", [(0, 1), (1, 2), (7, 2), (100_000_000, 8), (200_001, 3)])
def test_shard_slots_partition(n, world):
    """Round-robin sharding covers every slot exactly once (BASELINE.json.configs[4])."""
    from paper_1807_01527_b200.dist import shard_slots
    seen = []
    for r in range(world):
        j0, stride, m = shard_slots(n, r, world)
        assert stride == world and j0 == r
        if n <= 10_000_000:
            seen.extend(range(j0, n, stride)[:m])
        assert m == len(range(j0, n, stride))
    if n <= 10_000_000:
        assert sorted(seen) == list(range(n))
