"""CPU: the multi-GPU plumbing (shards + top-k all-gather merge) on world_size 2 with gloo."""
import os
import random

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1901_06229_b200.distributed import gather_topk, merge_hits, shard_bounds


def test_shard_bounds_cover_library():
    for n in (0, 1, 7, 10000):
        for world in (1, 2, 3, 8):
            b = [shard_bounds(n, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            assert max(h - l for l, h in b) - min(h - l for l, h in b) <= 1


def test_merge_orders_ties_by_index():
    parts = [[(0.9, 5, 1), (0.8, 2, 0)], [(0.9, 3, 7), (0.1, 9, 2)]]
    assert merge_hits(parts, 3) == [(0.9, 3, 7), (0.9, 5, 1), (0.8, 2, 0)]


def _worker(rank, world, port, scores, k, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_bounds(len(scores), world, rank)
    local = sorted(((scores[i], i, i % 32) for i in range(lo, hi)), key=lambda h: (-h[0], h[1]))[:k]
    merged = gather_topk(local, k, torch.device("cpu"))
    q.put((rank, merged))
    dist.destroy_process_group()


@pytest.mark.parametrize("n,k", [(1000, 100), (7, 10)])
def test_gather_topk_gloo_world2(n, k):
    rnd = random.Random(n)
    scores = [round(rnd.random(), 3) for _ in range(n)]  # coarse values -> plenty of exact ties
    want = sorted(((scores[i], i, i % 32) for i in range(n)), key=lambda h: (-h[0], h[1]))[:k]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + n % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, scores, k, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, merged in got:
        assert merged == want, rank


def test_library_ranges_equal_slices_of_the_library():
    """A rank generates its shard directly (make_library(first=, count=)): every ligand draws from
    its own stream (generate.cpp:76), so ranges are slices of the whole library."""
    import numpy as np
    import paper_1901_06229_b200 as gd
    spec = gd.LibrarySpec(3001, 40, 8, 0)
    full = gd.make_library(spec)
    for world in (1, 2, 3, 8):
        for r in range(world):
            lo, hi = shard_bounds(spec.count, world, r)
            part, want = gd.make_library(spec, first=lo, count=hi - lo), full.slice(lo, hi)
            for k in ("atom_off", "xyz", "radius", "bond_off", "bonds", "rot_off", "rots", "name_off"):
                assert np.array_equal(getattr(part, k), getattr(want, k)), (world, r, k)
            assert part.names == want.names


def test_bench_shards_strong_and_weak():
    import argparse
    import bench
    for scaling, base in (("strong", 10000), ("weak", 10000)):
        for world in (1, 2, 4, 8):
            args = argparse.Namespace(ligands=0, config="c2", scaling=scaling)
            parts = [bench.shard(args, world, r) for r in range(world)]
            total = parts[0][0]
            assert total == (base if scaling == "strong" else base * world)
            assert sum(c for _, _, c in parts) == total
            assert [f for _, f, _ in parts] == [sum(c for _, _, c in parts[:r]) for r in range(world)]
