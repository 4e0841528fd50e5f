"""Per-ligand device time of K1a / K1b against the batch size (tails of the persistent kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_06229_b200 as gd
ctx = gd.Context(0); ctx.set_pocket(gd.make_pocket()); ctx.set_params(gd.DockParams())
full = gd.make_library(gd.LibrarySpec(10000, 40, 8, 0))
for L in (625, 1250, 2500, 5000, 6875, 10000):
    b = ctx.stage(full.slice(0, L))
    for i in range(3):
        b.run(); ctx.sync(); ms = ctx.kernel_ms()
    print(L, "K1a us/lig %.3f  K1b us/lig %.3f" % (1e3 * ms["k1a_align"] / L, 1e3 * ms["k1b_sweep"] / L), flush=True)
    b.free()
