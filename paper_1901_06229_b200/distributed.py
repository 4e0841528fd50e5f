"""Multi-GPU plumbing for the screening path.

The library is cut into contiguous shards, one per rank (one process per GPU). Shards never talk
during the pose search: every DockResult is a pure function of (ligand, pocket, params), so
results are bit-identical for any shard count. The only exchange is the final top-k merge: each
rank's device top-k (K3) records are all-gathered once (NCCL on GPUs, gloo in the CPU tests) and
merged by (best_score desc, global ligand index asc).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist

Hit = Tuple[float, int, int]  # (best_score, global ligand index, best restart)


def shard_bounds(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous shard [lo, hi) of n ligands for `rank` (sizes differ by at most one)."""
    return n * rank // world, n * (rank + 1) // world


def merge_hits_array(parts: Sequence[np.ndarray], k: int) -> np.ndarray:
    """Global top-k from per-shard top-k record arrays ((m, 3) float64: score, global ligand index,
    restart; padding rows have index -1): ordered by (score desc, index asc), vectorised."""
    allh = np.concatenate([np.asarray(p, np.float64).reshape(-1, 3) for p in parts]) if parts else np.zeros((0, 3))
    allh = allh[allh[:, 1] >= 0]
    order = np.lexsort((allh[:, 1], -allh[:, 0]))[:k]
    return allh[order]


def merge_hits(parts: Sequence[Sequence[Hit]], k: int) -> List[Hit]:
    """Global top-k from per-shard top-k lists (each already ordered)."""
    arr = merge_hits_array([np.asarray(p, np.float64).reshape(-1, 3) for p in parts], k)
    return [(float(s), int(i), int(r)) for s, i, r in arr]


def gather_topk_array(local: np.ndarray, k: int, device: torch.device, group=None) -> np.ndarray:
    """All-gather every rank's local top-k records ((m, 3) float64 array: score, global index,
    restart; m <= k) and merge them: one collective of k x 3 doubles per rank (ranks with fewer
    than k records pad with index -1), the merge vectorised on the host. Indices < 2**53 and
    restarts are exact in float64."""
    world = dist.get_world_size(group)
    t = torch.full((k, 3), -1.0, dtype=torch.float64)
    m = min(k, len(local))
    if m:
        t[:m] = torch.from_numpy(np.ascontiguousarray(np.asarray(local, np.float64)[:m]))
    t = t.to(device)
    if device.type == "cuda":
        out = torch.empty((world * k, 3), dtype=torch.float64, device=device)
        dist.all_gather_into_tensor(out, t, group=group)
        allh = out.cpu().numpy()
    else:
        outs = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(outs, t, group=group)
        allh = torch.cat(outs).numpy()
    return merge_hits_array([allh], k)


def gather_topk(local: Sequence[Hit], k: int, device: torch.device, group=None) -> List[Hit]:
    """gather_topk_array for a list of (score, global index, restart) records."""
    arr = gather_topk_array(np.asarray(local, np.float64).reshape(-1, 3), k, device, group)
    return [(float(s), int(i), int(r)) for s, i, r in arr]
