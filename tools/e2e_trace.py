import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, paper_1901_06229_b200 as gd
lib = gd.make_library(gd.LibrarySpec(10000, 40, 8, 0))
ctx = gd.Context(0); ctx.set_pocket(gd.make_pocket()); ctx.set_params(gd.DockParams())
ctx.dock(lib)
for i in range(3):
    t = time.perf_counter(); ctx.dock(lib); print("e2e ms", round((time.perf_counter() - t) * 1e3, 2), flush=True)
