"""GPU: the multi-rank screening path with several ranks on one GPU (the driver's box has one).

Each rank is its own process with its own gd_ctx on cuda:0, docks its contiguous shard of one
library (generated directly as a range, make_library(first=, count=)), computes its device top-k
(K3) and joins the gloo all-gather of the top-k records (distributed.gather_topk), exactly as
bench.py's N-GPU step does with NCCL. The merged results must equal the single-process run for
2 and 4 ranks: every ligand's outputs bit for bit (acceptance #1's shard-count invariance,
acceptance_main.cpp:78-98) and the global top-k.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SPEC = dict(count=1500, atoms=40, rotamers=8, seed=0)
CLASH = 0.2  # commits live
K = 64


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, q):
    import paper_1901_06229_b200 as gd
    from paper_1901_06229_b200.distributed import gather_topk, shard_bounds
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_bounds(SPEC["count"], world, rank)
    lib = gd.make_library(gd.LibrarySpec(**SPEC), first=lo, count=hi - lo)
    with gd.Context(0) as ctx:
        ctx.set_pocket(gd.make_pocket())
        ctx.set_params(gd.DockParams(clash_factor=CLASH))
        b = ctx.stage(lib)
        b.run()
        out = b.fetch(trace=True)
        hits = [(s, i + lo, r) for s, i, r in b.topk(K)]
        b.free()
    merged = gather_topk(hits, K, torch.device("cpu"))
    parts = [None] * world
    dist.all_gather_object(parts, (lo, out.best_score, out.best_restart, out.final_xyz, out.step_k))
    if rank == 0:
        q.put((merged, parts))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_ranks_equal_one_rank(world):
    import paper_1901_06229_b200 as gd
    lib = gd.make_library(gd.LibrarySpec(**SPEC))
    with gd.Context(0) as ctx:
        one = ctx.dock(lib, gd.make_pocket(), gd.DockParams(clash_factor=CLASH), trace=True)
    order = np.lexsort((np.arange(lib.n_ligands), -one.best_score))[:K]
    want = [(float(one.best_score[i]), int(i), int(one.best_restart[i])) for i in order]

    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    port = _port()
    procs = [ctx_mp.Process(target=_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    merged, parts = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert merged == want
    parts.sort(key=lambda t: t[0])
    assert np.array_equal(np.concatenate([p[1] for p in parts]), one.best_score)
    assert np.array_equal(np.concatenate([p[2] for p in parts]), one.best_restart)
    assert np.array_equal(np.concatenate([p[3] for p in parts]), one.final_xyz)
    assert np.array_equal(np.concatenate([p[4] for p in parts]), one.step_k)
