"""Small cases for compute-sanitizer: C2-shape, clash 0.1 (commits), a mixed-size batch (every size
class + a >128-atom ligand) and C4 shape (NS = 4 incremental refresh)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_06229_b200 as gd
pocket = gd.make_pocket()
ctx = gd.Context(0)
p = gd.DockParams(n_restarts=4, clash_factor=0.1)
ctx.dock(gd.make_library(gd.LibrarySpec(6, 40, 8, 1)), pocket, p, trace=True)
ctx.dock(gd.make_library(gd.LibrarySpec(2, 120, 32, 2)), pocket, p, trace=True)
parts = [gd.make_library(gd.LibrarySpec(2, k, 4, 3)).slice(0, 1) for k in (20, 50, 90, 150)]
lib = gd.parse_library("".join(gd.serialize_library(x) for x in parts).encode())
ctx.dock(lib, pocket, gd.DockParams(n_restarts=4), trace=True)
print("sanitize cases ok")
