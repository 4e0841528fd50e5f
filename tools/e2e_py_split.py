"""Where the end-to-end time of Context.dock goes outside the executor (one C2 library, 10k)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import paper_1901_06229_b200 as gd
lib = gd.make_library(gd.LibrarySpec(10000, 40, 8, 0))
ctx = gd.Context(0)
ctx.set_pocket(gd.make_pocket())
ctx.set_params(gd.DockParams())
ctx.dock(lib)
for i in range(5):
    t0 = time.perf_counter()
    L, keep = lib._c()
    t1 = time.perf_counter()
    out, r = ctx._alloc_results(lib, False)
    t2 = time.perf_counter()
    rc = ctx._lib.gd_dock_batch(ctx._h, C.byref(L), C.byref(r))
    t3 = time.perf_counter()
    rt = ctx.run_times()
    print(f"_c {1e3*(t1-t0):.3f} alloc {1e3*(t2-t1):.3f} dock_batch {1e3*(t3-t2):.3f} busy {1e3*rt['busy']:.3f} total {1e3*(t3-t0):.3f}", flush=True)
    del out
