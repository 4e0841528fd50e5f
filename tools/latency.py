"""dock_ligand latency (one ligand through gd_dock_batch) and small-batch e2e times."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_06229_b200 as gd
pocket = gd.make_pocket(); p = gd.DockParams()
lib = gd.make_library(gd.LibrarySpec(64, 40, 8, 0))
ctx = gd.Context(0); ctx.set_pocket(pocket); ctx.set_params(p)
for L in (1, 1, 8, 64):
    sub = lib.slice(0, L)
    ctx.dock(sub)
    ts = []
    for i in range(5):
        t = time.perf_counter(); ctx.dock(sub); ts.append((time.perf_counter() - t) * 1e3)
    print(f"{L} ligands: e2e {min(ts):.2f} ms (min of 5)", {k: round(v * 1e3, 3) for k, v in ctx.run_times().items()}, flush=True)
