#!/usr/bin/env python3
"""Benchmark: GeoDock per-ligand pose search on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c1|c4|c5|c5s] [--scaling strong|weak] [--ligands L] [--backend nccl|gloo]

A "step" is one pass of the hot path over the synthetic library resident in HBM: the pose search
(K1a coarse alignment, K1b exact refinement + dihedral sweep, K2 best restart), the device top-k
(K3) and, for N > 1, the one exchange of the path: an all-gather of every rank's top-k records
(NCCL), merged into the global top-k. Ranks hold contiguous shards of one library:
  --scaling strong (default): the config's library (C2/C3: 10k ligands) split over N GPUs;
  --scaling weak: the config's library size per GPU (N x that in total).
`value` is ligands/s over all ranks, device-timed with CUDA events on the library's stream, max
over ranks, L2 flushed (256 MiB write) before every timed step. `e2e` is the same metric through
the public C-ABI call gd_dock_batch with host buffers (validation, packing, H2D, kernels, D2H)
plus the host top-k and the all-gather, wall-clocked per step, max over ranks.

With --gpus N > 1 and no torchrun environment, the script relaunches itself under
torch.distributed.run with N ranks (127.0.0.1). Ranks map to GPUs by LOCAL_RANK modulo the
visible device count; when ranks share a GPU the gather runs over gloo.

--impl reference times the reference's own CPU implementation (oracle/_ref: the unmodified
reference's run_screening, all host threads) on bounded samples of the same workload.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import struct
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json's metric, verbatim (the bench contract quotes it)
METRIC = "ligands/sec (device-timed, 1/2/4/8 B200) vs CPU ref; % of gather/FP32 roofline"

# name: (LibrarySpec kwargs, PocketSpec kwargs, f_in measured by the oracle,
#        CPU-reference sample, workload text)
C2_TEXT = "C2/C3: 10k synthetic ligands x 40 atoms x 8 rotamers vs one 24^3 (0.75 A) pocket"
CONFIGS = {
    "c1": (dict(count=100, atoms=32, rotamers=4), dict(), 0.8387, 100,
           "C1: 100 synthetic ligands x 32 atoms x 4 rotamers vs one 24^3 (0.75 A) pocket"),
    "c2": (dict(count=10000, atoms=40, rotamers=8), dict(), 0.8304, 256, C2_TEXT),
    "c3": (dict(count=10000, atoms=40, rotamers=8), dict(), 0.8304, 256, C2_TEXT),
    "c4": (dict(count=1000, atoms=120, rotamers=32), dict(), 0.8024, 64,
           "C4: 1k synthetic ligands x 120 atoms x 32 rotamers vs one 24^3 (0.75 A) pocket"),
    "c5": (dict(count=1000000, atoms=40, rotamers=8), dict(dims=(47, 47, 47), spacing=0.375), 0.8321, 256,
           "C5: 1M synthetic ligands x 40 atoms x 8 rotamers vs one 47^3 (0.375 A) pocket (L2-persistent cells)"),
    "c5s": (dict(count=10000, atoms=40, rotamers=8), dict(dims=(47, 47, 47), spacing=0.375), 0.8321, 256,
            "C5 grid, 10k sample: 10k ligands x 40 atoms x 8 rotamers vs one 47^3 (0.375 A) pocket"),
}
CPU_SAMPLE_1T = {"c1": 16, "c2": 16, "c3": 16, "c4": 4, "c5": 16, "c5s": 16}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def shard(args, world, rank):
    """(total ligands, first, count) of this rank (contiguous shards, distributed.shard_bounds)."""
    from paper_1901_06229_b200.distributed import shard_bounds
    base = args.ligands or CONFIGS[args.config][0]["count"]
    total = base * world if args.scaling == "weak" else base
    lo, hi = shard_bounds(total, world, rank)
    return total, lo, hi - lo


def config_dict(args, world):
    """The config both arms report (identical by construction)."""
    import paper_1901_06229_b200 as gd
    lspec, pspec, _, _, text = CONFIGS[args.config]
    total, _, _ = shard(args, world, 0)
    return {"workload": text, "ligands_total": total,
            "ligands_per_gpu": total if world == 1 else f"{total // world}-{-(-total // world)}",
            "atoms": lspec["atoms"], "rotamers": lspec["rotamers"],
            "pocket": {"dims": list(pspec.get("dims", (24, 24, 24))), "spacing": pspec.get("spacing", 0.75)},
            "params": gd.DockParams(clash_factor=args.clash).__dict__,
            "scaling": args.scaling if world > 1 else "n/a (1 GPU)",
            "l2": "flushed (256 MiB write) before every timed step", "topk": args.topk,
            "parallelism": (f"library sharded over {world} GPUs ({args.scaling} scaling), one top-k all-gather"
                            if world > 1 else "1 GPU")}


# ---------------------------------------------------------------------------- work model
def work_model(lib, params, f_in):
    """Algorithmic work of a library: the model's FP32 lane-ops and gathered bytes.
    Generated ligands are trees (generate.cpp:83-103): the moving set of rotamer (p, c) is the
    subtree of c, children have larger indices than their parents."""
    N, G = params.n_restarts, int(np.prod(params.rotation_steps))
    reps, S = params.num_repetitions, params.dihedral_steps
    L = lib.n_ligands
    n = int(lib.atom_off[1] - lib.atom_off[0]) if L else 0
    assert np.all(np.diff(lib.atom_off) == n), "work model expects one ligand shape"
    R = int(lib.rot_off[1] - lib.rot_off[0]) if L else 0
    par = lib.bonds.reshape(L, n - 1, 2)[:, :, 0].astype(np.int64)  # parent of atom e + 1
    size = np.ones((L, n), np.int64)
    rows = np.arange(L)
    for a in range(n - 1, 0, -1):
        np.add.at(size, (rows, par[:, a - 1]), size[:, a])
    j = lib.rots.reshape(L, R, 2)[:, :, 1].astype(np.int64)
    m = np.take_along_axis(size, j, axis=1)  # |moving set| per rotamer
    w_align = N * G * n * L
    w_sweep = int(N * reps * (S - 1) * (m - 1).sum())
    p_cross = int(N * reps * (S - 1) * ((m - 1) * (n - m)).sum())
    W = w_align + w_sweep
    return dict(w_align=w_align, w_sweep=w_sweep, p_cross=p_cross, fp32_ops=W * (15 + 21 * f_in) + 7 * p_cross,
                gather_bytes=32 * f_in * W)


def fp32_peak_per_clk():
    """FFMA lane-ops per clock per SM measured by tools/fp32_peak.cu (profiles/fp32_peak.json),
    else the nominal 128 (4 SM sub-partitions x 32 FP32 lanes)."""
    p = os.path.join(ROOT, "profiles", "fp32_peak.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["ffma_lane_ops_per_clk_per_sm"]), "measured (tools/fp32_peak.cu, profiles/fp32_peak.json)"
    return 128.0, "nominal"


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for k, v in zip(names, r[3:7]):
                if v.lower() == "active":
                    reasons.add(k)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------- CPU reference
def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_reference(args, steps):
    """The reference's run_screening (pipeline.cpp:187-290, n_devices = 0) on the host cores, on the
    first `sample` ligands of the same library: all host threads, median over
    `steps` runs, plus one single-thread (n_workers = 1) run on a smaller prefix."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle, Params
    ref = Oracle("reference")
    lspec, pspec, _, sample, _ = CONFIGS[args.config]
    sample = args.cpu_sample or sample
    nproc = host_threads()
    pocket = ref.make_pocket(**pspec) if pspec else ref.make_pocket()
    lib = ref.make_library(sample, lspec["atoms"], lspec["rotamers"], 0)
    p = Params(clash_factor=args.clash)
    vals = []
    for _ in range(max(1, steps)):
        _, _, wall = ref.run_screening(lib, pocket, p, n_workers=nproc)
        vals.append(sample / wall)
    s1 = CPU_SAMPLE_1T[args.config]
    lib1 = ref.make_library(s1, lspec["atoms"], lspec["rotamers"], 0)
    _, _, wall1 = ref.run_screening(lib1, pocket, p, n_workers=1)
    return {"value": round(statistics.median(vals), 3), "unit": "ligands/s", "cores": nproc, "kind": "reference",
            "sample": f"first {sample} ligands of the same library per run, unmodified reference run_screening "
                      f"(oracle/_ref, n_devices = 0), {nproc} workers, median of {len(vals)} runs",
            "runs": [round(v, 3) for v in vals],
            "single_thread": {"value": round(s1 / wall1, 3), "unit": "ligands/s", "cores": 1,
                              "sample": f"first {s1} ligands, n_workers = 1"},
            "cpu_model": cpu_model(), "nproc": os.cpu_count()}


# ---------------------------------------------------------------------------- our arm
def topk_digest(hits):
    h = hashlib.sha256()
    for s, i, r in hits:
        h.update(struct.pack("<dQI", s, i, r))
    return h.hexdigest()[:16]


def host_topk(score, k):
    """Indices of the k best ligands by (score desc, index asc), as the device top-k (K3) orders
    them: a partition picks every ligand scoring at least the k-th best, a sort orders those."""
    n = len(score)
    k = min(k, n)
    if k == 0:
        return np.zeros(0, np.int64)
    cand = np.arange(n)
    if k < n:
        kth = np.partition(-score, k - 1)[k - 1]
        cand = np.flatnonzero(-score <= kth)
    return cand[np.lexsort((cand, -score[cand]))][:k]


def run_ours(args):
    import torch
    import paper_1901_06229_b200 as gd
    from paper_1901_06229_b200.distributed import gather_topk_array

    rank, world, local = dist_env()
    n_dev = max(1, torch.cuda.device_count())
    dev = local % n_dev
    torch.cuda.set_device(dev)
    backend = args.backend or ("nccl" if world <= n_dev else "gloo")  # NCCL needs one GPU per rank
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    gdev = torch.device("cuda", dev) if backend == "nccl" else torch.device("cpu")

    lspec, pspec, f_in, _, _ = CONFIGS[args.config]
    total, first, count = shard(args, world, rank)
    params = gd.DockParams(clash_factor=args.clash)
    pocket = gd.make_pocket(gd.PocketSpec(**pspec))
    lib = gd.make_library(gd.LibrarySpec(total, lspec["atoms"], lspec["rotamers"], 0), first=first, count=count)
    mode = gd.MODE_EXACT if args.exact else gd.MODE_FAST
    ctx = gd.Context(dev, mode=mode | (gd.FLAG_SKIP_INVARIANT_CLASH if args.skip_invariant else 0))
    ctx.set_pocket(pocket)
    ctx.set_params(params)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    topk = args.topk

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(vals):
        if dist is None:
            return vals
        t = torch.tensor(vals, dtype=torch.float64, device=gdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    def sum_over_ranks(vals):
        if dist is None:
            return vals
        t = torch.tensor(vals, dtype=torch.float64, device=gdev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t.tolist()

    def timed(batch, steps, warmup, clocks=None):
        """Device time (ms) of `steps` steps (kernels + top-k + all-gather), L2 flushed before each,
        the per-kernel event times of the last gd_run, and the merged global top-k."""
        def step():
            batch.run()
            hits = batch.topk_array(topk)  # K3 + D2H of k records (score, index, restart)
            hits[:, 1] += first            # global ligand indices
            if dist is not None:  # the one exchange of the path: all-gather of the top-k records
                with torch.cuda.stream(stream):
                    hits = gather_topk_array(hits, topk, gdev)
            return hits

        for _ in range(warmup):
            step()
        torch.cuda.synchronize(dev)
        barrier()
        times, kms = [], []
        for _ in range(steps):
            with torch.cuda.stream(stream):
                flush.fill_(1)  # L2 flush (256 MiB > 126 MB L2), outside the timed region
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            hits = step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
            kms.append(ctx.kernel_ms())
        k1a = statistics.mean(k["k1a_align"] for k in kms)
        k1b = statistics.mean(k["k1b_sweep"] for k in kms)
        k2 = statistics.mean(k["k2_finalize"] for k in kms)
        ms, k1a, k1b, k2 = max_over_ranks([statistics.mean(times), k1a, k1b, k2])
        return ms, k1a, k1b, k2, [(float(s), int(i), int(r)) for s, i, r in hits]

    sm_hz_guess = 1965e6
    per_clk, peak_src = fp32_peak_per_clk()

    def roof(st, k1a_ms, k1b_ms, sm_mhz):
        """FP32 lane-op roofline on the work each kernel executed (device counters, summed over ranks)."""
        peak = 148 * per_clk * sm_mhz * 1e6 / 1e12
        peak_nominal = 148 * 128 * sm_mhz * 1e6 / 1e12
        w_align = params.n_restarts * int(np.prod(params.rotation_steps)) * lspec["atoms"] * total
        ops_a = w_align * (15 + 21 * f_in)
        ops_b = st["sweep_samples"] * (15 + 21 * f_in) + 7 * st["cross_pairs"]
        gpus = min(world, n_dev)  # per-GPU rate (ranks sharing one GPU in the gloo tests share its peak)
        a = ops_a / (k1a_ms / 1e3) / 1e12 / gpus
        b = ops_b / (k1b_ms / 1e3) / 1e12 / gpus if k1b_ms > 0 else 0.0
        pth = (ops_a + ops_b) / ((k1a_ms + k1b_ms) / 1e3) / 1e12 / gpus
        return dict(peak=peak, peak_nominal=peak_nominal, ops_a=ops_a, ops_b=ops_b, a=a, b=b, path=pth)

    # ---- headline: the configured regime
    batch = ctx.stage(lib)
    with ClockSampler(dev) as clocks:
        ms, k1a_ms, k1b_ms, k2_ms, hits = timed(batch, args.steps, args.warmup)
    st_local = ctx.stats()
    launches_per_step = st_local["launches"] + 2  # gd_run's kernels + topk prepare/emit (cub sorts not counted)
    keys = ["sweep_steps", "sweep_invariant_steps", "sweep_scored_steps", "sweep_samples", "cross_pairs",
            "restarts", "commits", "step_exact_evals", "align_exact_evals", "align_fallbacks", "step_fallbacks",
            "align_second_passes"]
    st = dict(zip(keys, (int(v) for v in sum_over_ranks([float(st_local[k]) for k in keys]))))
    chk = batch.fetch()
    batch.free()

    # ---- e2e through the public C-ABI (host buffers in and out) + host top-k + all-gather
    e2e_times = []
    res = None
    for it in range(max(1, min(args.steps, 3)) + 1):
        torch.cuda.synchronize(dev)
        barrier()
        t0 = time.perf_counter()
        res = ctx.dock(lib)
        order = host_topk(res.best_score, topk)
        e2e_hits = np.stack([res.best_score[order], (order + first).astype(np.float64),
                             res.best_restart[order].astype(np.float64)], axis=1)
        if dist is not None:
            e2e_hits = gather_topk_array(e2e_hits, topk, gdev)
        t1 = time.perf_counter()
        if it > 0:
            e2e_times.append(t1 - t0)
    e2e_s = max_over_ranks([statistics.mean(e2e_times)])[0]
    e2e_stats = ctx.stats()
    h2d = int(sum_over_ranks([float(e2e_stats.get("h2d_bytes", 0))])[0])
    d2h = int(sum_over_ranks([float(e2e_stats.get("d2h_bytes", 0))])[0])
    assert np.array_equal(chk.best_score, res.best_score), "staged vs e2e results differ"
    e2e_hits = [(float(s), int(i), int(r)) for s, i, r in e2e_hits]
    assert e2e_hits == hits, "e2e top-k differs from the device top-k"

    # ---- sweep regimes beside the headline (1 GPU): the live-commit sweep at clash 0.1 and the
    # invariant-clash skip (reported separately from the headline)
    regimes = {}
    if world == 1 and not args.no_regimes and not args.exact:
        for name, clash, flags in (("clash_0.1", 0.1, 0), ("skip_invariant", args.clash, gd.FLAG_SKIP_INVARIANT_CLASH)):
            ctx.set_mode(mode | flags)
            ctx.set_params(gd.DockParams(clash_factor=clash))
            b2 = ctx.stage(lib)
            r_ms, r_a, r_b, _, _ = timed(b2, max(1, min(args.steps, 3)), 1)
            rs = ctx.stats()
            b2.free()
            rr = roof(rs, r_a, r_b, clocks.summary()["sm_mhz"] or sm_hz_guess / 1e6)
            regimes[name] = {"clash_factor": clash, "skip_invariant_clash": bool(flags),
                             "value": round(total / (r_ms / 1e3), 2), "ms_per_step": round(r_ms, 3),
                             "k1a_ms": round(r_a, 3), "k1b_ms": round(r_b, 3),
                             "k1a_frac": round(rr["a"] / rr["peak"], 4), "k1b_frac": round(rr["b"] / rr["peak"], 4),
                             "path_frac": round(rr["path"] / rr["peak"], 4),
                             "stats": {k: int(rs[k]) for k in keys}}
        ctx.set_mode(mode)
        ctx.set_params(params)

    clock = clocks.summary()
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    value = total / (ms / 1e3)
    sm_mhz = clock["sm_mhz"] or sm_hz_guess / 1e6
    rr = roof(st, k1a_ms, k1b_ms, sm_mhz)
    # the faithful model (every cross pair of every step) for comparison: computed on
    # up to 20k ligands of rank 0's shard and scaled to the library (one ligand shape throughout)
    wm_sub = lib.slice(0, min(count, 20000))
    wm = {k: v * total / wm_sub.n_ligands for k, v in work_model(wm_sub, params, f_in).items()}
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tpath) and world == 1 and total == lspec["count"]:
        traffic = json.load(open(tpath)).get("k1a_dram_bytes_per_launch")
    line = {
        "metric": METRIC,
        "value": round(value, 2), "unit": "ligands/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": args.scaling if world > 1 else "strong",
        "vs_baseline": None, "dtype": "f32 coarse + f64 exact", "data": "synthetic (reference generator, seed 0)",
        "impl": "ours", "mode": ("exact" if args.exact else "fast") + ("+skip_invariant" if args.skip_invariant else ""),
        "backend": backend if world > 1 else None,
        "config": config_dict(args, world),
        "e2e": {"value": round(total / e2e_s, 2), "unit": "ligands/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "what": "gd_dock_batch (validate, pack, H2D, kernels, D2H) + top-k gather"},
        "gpu_launches": launches_per_step,
        "roofline": {
            "bound": "fp32", "achieved": round(rr["a"], 3), "peak": round(rr["peak"], 3), "unit": "TFLOP/s",
            "frac": round(rr["a"] / rr["peak"], 4), "traffic": traffic,
            "kernel": "K1a coarse alignment (dominant), FP32 lane-ops per GPU",
            "k1a_ms": round(k1a_ms, 4),
            "k1b": {"kernel": "K1b exact refinement + dihedral sweep (executed work: device counters)",
                    "ms": round(k1b_ms, 4), "achieved": round(rr["b"], 3), "frac": round(rr["b"] / rr["peak"], 4)},
            "k2_ms": round(k2_ms, 4),
            "path": {"kernels": "K1a + K1b", "ms": round(k1a_ms + k1b_ms, 4), "achieved": round(rr["path"], 3),
                     "frac": round(rr["path"] / rr["peak"], 4)},
            "peak_source": f"148 SM x {per_clk:.1f} FFMA lane-ops/clk ({peak_src}) x {sm_mhz:.0f} MHz "
                           f"(median SM clock under load)",
            "frac_vs_nominal_128": round(rr["a"] / rr["peak_nominal"], 4),
            "executed_work": {"k1a_lane_ops": rr["ops_a"], "k1b_lane_ops": rr["ops_b"], "f_in": f_in,
                              "model": "sample = 15 + 21 f_in lane-ops, cross pair = 7 (SURVEY §8(d))"},
            "work_model_faithful": wm,
        },
        "sweep": st,
        "regimes": regimes or None,
        "topk_digest": topk_digest(hits), "topk_best": list(hits[0]) if hits else None,
        "clocks": clock,
    }
    if not args.no_cpu and world == 1:
        line["cpu_baseline"] = cpu_reference(args, 3)
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cb = cpu_reference(args, args.steps)
    v = cb["value"]
    line = {"metric": METRIC, "value": v, "unit": "ligands/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 / v * (args.cpu_sample or CONFIGS[args.config][3]), 3),
            "higher_is_better": True, "scaling": args.scaling if world > 1 else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference generator, seed 0)",
            "impl": "reference", "config": config_dict(args, world), "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "ligands/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def relaunch(args):
    """--gpus N > 1 outside torchrun: re-exec under torch.distributed.run with N ranks."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--ligands", type=int, default=0, help="library size (strong) / per GPU (weak); default: the config's")
    ap.add_argument("--clash", type=float, default=0.75)
    ap.add_argument("--topk", type=int, default=100)
    ap.add_argument("--backend", default=None, choices=["nccl", "gloo"], help="default: nccl, gloo if ranks share a GPU")
    ap.add_argument("--exact", action="store_true", help="GD_MODE_EXACT kernel (FP64 everywhere)")
    ap.add_argument("--skip-invariant", action="store_true", help="GD_FLAG_SKIP_INVARIANT_CLASH (reported separately)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-regimes", action="store_true", help="skip the clash-0.1 / skip-invariant sub-measurements")
    ap.add_argument("--cpu-sample", type=int, default=0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
