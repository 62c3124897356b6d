"""Host-side multi-GPU logic of the ASSE hot path.

Packets of a slice are split round-robin across ranks: slot j goes to rank
j mod D (BASELINE.json.configs[4]). Every rank scans its shard into a local
per-slice touch bitmap; at end_slice the bitmaps are OR-merged over NVLink peer
memory (k_merge_or, csrc/asse_kernels.cu) so every rank folds the same global
touches into an identical replicated AT pool (A26 combine rule).
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
