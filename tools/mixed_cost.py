"""Cost of a mixed batch: the C2 library alone vs the C2 library plus one 70-atom ligand (NS = 4
kernels for everything) vs plus one 150-atom ligand (routed to the FP64 kernel)."""
import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_06229_b200 as gd
base = gd.make_library(gd.LibrarySpec(4000, 40, 8, 0))
txt = gd.serialize_library(base)
libs = {"c2": gd.parse_library(txt.encode())}
for extra in (70, 150):
    e = gd.make_library(gd.LibrarySpec(1, extra, 8, 9))
    libs[f"c2+{extra}"] = gd.parse_library((txt + gd.serialize_library(e)).encode())
ctx = gd.Context(0); ctx.set_pocket(gd.make_pocket()); ctx.set_params(gd.DockParams())
for k, lib in libs.items():
    b = ctx.stage(lib)
    for i in range(3):
        b.run(); ctx.sync(); ms = ctx.kernel_ms()
    print(k, {a: round(v, 2) for a, v in ms.items()}, flush=True)
    b.free()
