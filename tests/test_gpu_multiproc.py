"""libasse's own N>1 control path in two processes on ONE GPU.

Each process is one rank (gloo process group on 127.0.0.1): its context has world = 2,
its touch / merged / exchange buffers are CUDA IPC allocations whose handles are
exchanged over the group (dist.IpcPeers), and end_slice runs the eager multi-rank
sequence itself — barrier, k_merge_or / k_merge_shard over the peer buffers, fold,
restore with the exchange publication, barrier, k_gather_peers — with sync_mode 2
(host barriers through torch.distributed). No kernel waits on another rank's kernel,
so two ranks may share the GPU (B200_PROFILING.md: spinning kernels of several ranks on
one GPU are not safe; the device barrier itself is checked as one cooperative kernel
below). Every rank must produce the oracle's reports and pool (its frames in option S)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, shard, name, N, T, variant, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from gen import PRESETS, Generator
        from oracle import oracle as O
        from paper_1807_01527_b200 import asse
        from paper_1807_01527_b200.dist import IpcPeers, shard_slots
        from parity import compare_pool, compare_reports

        p = dict(PRESETS[name])
        ctx = asse.Asse(**dict(p, world=world, rank=rank, frame_shard=shard))
        ctx.set_scan_variant(variant)
        peers = IpcPeers(ctx)
        ora = O.Oracle(**p)
        g = Generator(name, N=N)
        F = 1 << p["u"]
        for t in range(T):
            j0, stride, n = shard_slots(g.N, rank, world)
            mine = g.slice(t, j0=j0, stride=stride, n=n)
            d = torch.from_numpy(mine.view(np.int32).reshape(-1)).cuda()
            ctx.scan_slice(d)
            rep = ctx.end_slice(1)
            ora.scan(g.slice(t))
            ro = ora.end_slice(1)
            compare_reports(rep, ro, p["theta"], "rank %d t=%d" % (rank, t))
            pool = ora.pool()
            if shard:
                Fl = F // world
                pool = pool[:, rank * Fl:(rank + 1) * Fl]
            compare_pool(ctx.pool(), pool, "rank %d t=%d" % (rank, t))
        st = ctx.stats()
        assert st["host_barriers"] == 2 * T, st["host_barriers"]
        dist.barrier()
        ctx.close()
        peers.close()
        q.put((rank, True))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("shard", [0, 1])
@pytest.mark.parametrize("name,N,T,variant", [("C3", 1_500_000, 3, 3), ("C1", None, 4, 0)])
def test_two_processes_one_gpu_ipc_host_barrier(cuda_device, shard, name, N, T, variant):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, shard, name, N, T, variant, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res


@pytest.mark.parametrize("world", [2, 3, 8, 16])
def test_device_barrier_protocol_cooperative(cuda_device, world):
    """k_barrier's release/acquire protocol (sync_mode 0) with the ranks played by the
    blocks of one cooperative launch: after every barrier each rank sees every rank's
    data of that epoch, and no rank overwrites data a peer has not read yet."""
    from paper_1807_01527_b200 import asse
    assert asse.selftest_barrier(world, 2000) == 0


@pytest.mark.parametrize("extra", [[], ["--replicated"]])
def test_bench_two_ranks_one_device(cuda_device, extra):
    """bench.py's N>1 path (round-robin shards, frame-sharded or replicated pools, the
    library's multi-rank end_slice, max-over-ranks timing, rank-0 JSON line) launched as the
    driver launches it (torch.distributed.run), with both ranks on cuda:0 through CUDA IPC
    peers and host barriers (--one-device). The numbers of such a run mean nothing."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(root, "bench.py"), "--gpus", "2", "--one-device", "--workload", "C3",
           "--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu", "--distinct", "4"] + extra
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    assert "IPC" in d["config"]["peers"]
    assert d["config"]["parallelism"].startswith("dp2")
    assert d["reports_per_step"] > 0
