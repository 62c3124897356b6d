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
