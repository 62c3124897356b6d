"""Host-side multi-GPU logic of the ASSE hot path.

Packets of a slice are split round-robin across ranks: slot j goes to rank
j mod D (BASELINE.json.configs[4]). Every rank scans its shard into a local
per-slice touch bitmap; at end_slice the bitmaps are OR-merged over NVLink peer
memory (k_merge_or / k_merge_shard, csrc/asse_kernels.cuh; A26 combine rule).
Peer setup: attach_symmetric_peers (torch symmetric memory, device barrier,
sync_mode 0), IpcPeers (CUDA IPC handles over the process group, host barrier,
sync_mode 2) or attach_local_peers (virtual ranks in one process, sync_mode 1).
"""


def shard_slots(n_total, rank, world):
    """Slots j = rank, rank + world, ... of a slice of n_total packets.
    Returns (j0, stride, n_local)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    n_local = (n_total - rank + world - 1) // world if n_total > rank else 0
    return rank, world, n_local


def attach_symmetric_peers(ctx, group=None):
    """Allocate this rank's touch / merged bitmaps and signal pad in torch symmetric
    memory (NVLink peer-mapped), exchange the peer pointers and hand them to the
    library (asse_attach_peers, sync_mode 0: device barrier over the signal pads).
    Returns the tensors (they must outlive ctx)."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem

    group = group or dist.group.WORLD
    dev = torch.device("cuda", torch.cuda.current_device())
    enable = getattr(symm_mem, "enable_symm_mem_for_group", None)
    if enable is not None:
        try:
            enable(group.group_name)
        except Exception:  # newer torch: no per-group opt-in needed
            pass
    shard = bool(ctx.cfg.frame_shard)
    sizes = [ctx.bitmap_bytes(), ctx.merged_bytes(), 256] + ([ctx.exchange_bytes()] if shard else [])
    bufs, ptrs = [], []
    for size in sizes:
        t = symm_mem.empty(size, dtype=torch.uint8, device=dev)
        t.zero_()
        h = symm_mem.rendezvous(t, group)
        bufs.append((t, h))
        ptrs.append(list(h.buffer_ptrs))
    torch.cuda.synchronize()
    dist.barrier(group)
    ctx.attach_peers(ptrs[0], ptrs[1], ptrs[2], ptrs[3] if shard else None, sync_mode=0)
    return bufs


def attach_local_peers(ctxs):
    """Single-GPU 'virtual ranks' (tests): every context gets plain device buffers
    and the caller orders the phases (sync_mode 1): scan all ranks, then
    ctx.merge() for every rank, synchronize, (frame_shard: end_slice_begin for every
    rank, synchronize,) then end_slice for every rank."""
    import torch
    shard = bool(ctxs[0].cfg.frame_shard)
    touch = [torch.zeros(c.bitmap_bytes(), dtype=torch.uint8, device="cuda") for c in ctxs]
    merged = [torch.zeros(c.merged_bytes(), dtype=torch.uint8, device="cuda") for c in ctxs]
    xchg = [torch.zeros(c.exchange_bytes(), dtype=torch.uint8, device="cuda") for c in ctxs] if shard else []
    tp = [t.data_ptr() for t in touch]
    mp = [t.data_ptr() for t in merged]
    xp = [t.data_ptr() for t in xchg] if shard else None
    torch.cuda.synchronize()
    for c in ctxs:
        c.attach_peers(tp, mp, None, xp, sync_mode=1)
    return touch, merged, xchg


class IpcPeers:
    """Peer buffers shared by CUDA IPC (one process per rank on one node) with the host
    barrier of sync_mode 2 (asse_set_host_barrier -> torch.distributed.barrier). Ranks may
    share a GPU: no kernel waits on another rank's kernel. Keep the object alive as long
    as the context; close() unmaps and frees the buffers."""

    def __init__(self, ctx, group=None, device=None):
        import torch
        import torch.distributed as dist
        from paper_1807_01527_b200 import asse

        group = group or dist.group.WORLD
        self.group = group
        dev = torch.cuda.current_device() if device is None else device
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        shard = bool(ctx.cfg.frame_shard)
        sizes = [ctx.bitmap_bytes(), ctx.merged_bytes()] + ([ctx.exchange_bytes()] if shard else [])
        self.own, self.opened, ptrs = [], [], []
        for size in sizes:
            p, h = asse.ipc_alloc(size, dev)
            self.own.append(p)
            handles = [None] * world
            dist.all_gather_object(handles, h, group=group)
            row = []
            for w in range(world):
                if w == rank:
                    row.append(p)
                else:
                    q = asse.ipc_open(handles[w], dev)
                    self.opened.append(q)
                    row.append(q)
            ptrs.append(row)
        dist.barrier(group)
        ctx.set_host_barrier(lambda: dist.barrier(group))
        ctx.attach_peers(ptrs[0], ptrs[1], None, ptrs[2] if shard else None, sync_mode=2)
        self.ptrs = ptrs

    def close(self):
        """Collective: unmap the peers' buffers, wait for every rank to do the same, then
        free this rank's own (the context using them must be destroyed first)."""
        import torch.distributed as dist
        from paper_1807_01527_b200 import asse
        for q in self.opened:
            asse.ipc_free(q, True)
        dist.barrier(self.group)
        for p in self.own:
            asse.ipc_free(p, False)
        self.opened, self.own = [], []
