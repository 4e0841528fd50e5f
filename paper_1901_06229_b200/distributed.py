"""Multi-GPU plumbing for the screening path.

The library is cut into contiguous shards, one per rank (one process per GPU). Shards never talk
during the pose search: every DockResult is a pure function of (ligand, pocket, params), so
results are bit-identical for any shard count. The only exchange is the final top-k merge: each
rank's device top-k (K3) records are all-gathered once (NCCL on GPUs, gloo in the CPU tests) and
merged by (best_score desc, global ligand index asc).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import torch
import torch.distributed as dist

Hit = Tuple[float, int, int]  # (best_score, global ligand index, best restart)


def shard_bounds(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous shard [lo, hi) of n ligands for `rank` (sizes differ by at most one)."""
    return n * rank // world, n * (rank + 1) // world


def merge_hits(parts: Sequence[Sequence[Hit]], k: int) -> List[Hit]:
    """Global top-k from per-shard top-k lists (each already ordered)."""
    allh = [tuple(h) for p in parts for h in p]
    allh.sort(key=lambda h: (-h[0], h[1]))
    return [(float(s), int(i), int(r)) for s, i, r in allh[:k]]


def gather_topk(local: Sequence[Hit], k: int, device: torch.device, group=None) -> List[Hit]:
    """All-gather every rank's local top-k records (global indices) and merge them.

    Records travel as float64 triples; ligand indices < 2**53 and restarts are exact in float64.
    Ranks may hold fewer than k records (small shards): each rank pads to k with sentinel rows.
    """
    world = dist.get_world_size(group)
    t = torch.full((k, 3), -1.0, dtype=torch.float64, device=device)
    if local:
        t[: len(local)] = torch.tensor([[s, i, r] for s, i, r in local[:k]], dtype=torch.float64, device=device)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    parts = [[(float(a), int(b), int(c)) for a, b, c in o.cpu().tolist() if b >= 0] for o in out]
    return merge_hits(parts, k)
