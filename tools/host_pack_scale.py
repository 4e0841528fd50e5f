"""Host half of the executor (validate + SoA pack, gd_host_pack) at 8-GPU concurrency, no GPU needed.

VERDICT r1 "next" #5: an 8-GPU end-to-end screen needs ~8 x 215k ligands/s of host packing. Three
ways of driving it, each packing 8 shards of a C2-shape library (10k ligands x 40 atoms x 8 rotamers
per shard):
  single   one caller, all host threads, the 8 shards one after another
  threads  8 concurrent callers in one process (run_screening's one-thread-per-device shape), each
           with its context-sized share of the host threads (nproc / 8)
  procs    8 processes (the torchrun shape, one per GPU), each with nproc / 8 threads
Aggregate = 8 x 10k ligands / the slowest caller's packing time (gd_host_pack's own clock: the
staging buffer and the host pool exist before it starts, as in the executor, which reuses both);
the wall time including that setup is reported beside it.
usage: python tools/host_pack_scale.py [--shards 8] [--ligands 10000] > profiles/r2_host_pack.json
"""
import argparse
import json
import multiprocessing as mp
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_06229_b200 as gd  # noqa: E402


def shard_lib(i, n, shards=8):
    """Shard i of an (shards x n)-ligand C2-shape library (every ligand has its own random stream)."""
    return gd.make_library(gd.LibrarySpec(shards * n, 40, 8, 0), first=i * n, count=n)


def _proc(i, n, threads, barrier, q):
    lib, pocket = shard_lib(i, n), gd.make_pocket(gd.PocketSpec())
    gd.host_pack_seconds(lib, pocket, threads=threads)  # warm (page faults, pool start)
    barrier.wait()
    t0 = time.time()
    s = gd.host_pack_seconds(lib, pocket, threads=threads)
    q.put((t0, time.time(), s))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shards", type=int, default=8)
    ap.add_argument("--ligands", type=int, default=10000)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    S, n, ncpu = a.shards, a.ligands, os.cpu_count()
    per = max(1, ncpu // S)
    pocket = gd.make_pocket(gd.PocketSpec())
    libs = [shard_lib(i, n) for i in range(S)]
    out = {"what": "gd_host_pack (validate + SoA pack of the executor) throughput, C2-shape shards",
           "nproc": ncpu, "shards": S, "ligands_per_shard": n,
           "cpu_model": next((l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")), "?")}

    best = 1e30
    for _ in range(a.reps):
        t = sum(gd.host_pack_seconds(l, pocket, threads=ncpu) for l in libs)
        best = min(best, t)
    out["single"] = {"threads": ncpu, "seconds": best, "ligands_per_s": S * n / best}

    for l in libs:
        gd.host_pack_seconds(l, pocket, threads=per)
    best = 1e30
    for _ in range(a.reps):
        res = [0.0] * S
        bar = threading.Barrier(S)

        def run(i):
            bar.wait()
            res[i] = gd.host_pack_seconds(libs[i], pocket, threads=per)

        th = [threading.Thread(target=run, args=(i,)) for i in range(S)]
        t0 = time.perf_counter()
        for t in th:
            t.start()
        for t in th:
            t.join()
        wall = time.perf_counter() - t0
        if max(res) < best:
            best, best_wall = max(res), wall
    out["threads"] = {"callers": S, "threads_each": per, "seconds": best, "ligands_per_s": S * n / best,
                      "wall_with_setup_s": best_wall}

    ctx = mp.get_context("spawn")
    best = 1e30
    for _ in range(a.reps):
        bar, q = ctx.Barrier(S), ctx.Queue()
        ps = [ctx.Process(target=_proc, args=(i, n, per, bar, q)) for i in range(S)]
        for p in ps:
            p.start()
        r = [q.get() for _ in range(S)]
        for p in ps:
            p.join()
        if max(x for _, _, x in r) < best:
            best, best_wall = max(x for _, _, x in r), max(e for _, e, _ in r) - min(s for s, _, _ in r)
    out["procs"] = {"processes": S, "threads_each": per, "seconds": best, "ligands_per_s": S * n / best,
                    "wall_with_setup_s": best_wall}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
