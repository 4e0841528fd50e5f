"""Profiling driver: stage a synthetic library and launch the pose search a few times (for ncu)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_06229_b200 as gd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ligands", type=int, default=1000)
ap.add_argument("--atoms", type=int, default=40)
ap.add_argument("--rotamers", type=int, default=8)
ap.add_argument("--clash", type=float, default=0.75)
ap.add_argument("--runs", type=int, default=2)
ap.add_argument("--exact", action="store_true")
ap.add_argument("--dims", type=int, default=24)
ap.add_argument("--spacing", type=float, default=0.75)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
ctx = gd.Context(0, mode=gd.MODE_EXACT if a.exact else gd.MODE_FAST)
ctx.set_pocket(gd.make_pocket(gd.PocketSpec(dims=(a.dims,) * 3, spacing=a.spacing)))
ctx.set_params(gd.DockParams(clash_factor=a.clash, num_repetitions=a.reps))
b = ctx.stage(gd.make_library(gd.LibrarySpec(a.ligands, a.atoms, a.rotamers, 0)))
import time
for i in range(a.runs):
    ctx.sync()
    t0 = time.perf_counter()
    b.run()
    ctx.sync()
    dt = time.perf_counter() - t0
    km = ctx.kernel_ms()
    print(f"run {i}: {dt*1e3:.2f} ms  {a.ligands/dt:.0f} lig/s  K1a {km['k1a_align']:.2f} K1b {km['k1b_sweep']:.2f} K2 {km['k2_finalize']:.2f} ms")
res = b.fetch()
print("mean best", float(res.best_score.mean()), ctx.stats())
