"""Ligand ingest throughput: gd_parse_library (multi-threaded C++) vs the reference's
parse_ligand_library (io.cpp:96-140, oracle/_ref), on the same serialized synthetic library.
Prints one JSON line. Host-only (no GPU)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_1901_06229_b200 as gd  # noqa: E402
from oracle import Oracle  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
lib = gd.make_library(gd.LibrarySpec(n, 40, 8, 0))
text = gd.serialize_library(lib).encode()
t0 = time.perf_counter()
ours = gd.parse_library(text)
t1 = time.perf_counter()
ref = Oracle("reference")
sample = min(n, 20_000)
cut = int(ours.atom_off[sample])  # bounded sample for the reference arm: the first `sample` records
sub = gd.serialize_library(ours.slice(0, sample)).encode()
t2 = time.perf_counter()
ref.parse_library(sub)
t3 = time.perf_counter()
print(json.dumps({"workload": f"{n} ligands x 40 atoms x 8 rotamers, .lgd text ({len(text) / 1e6:.1f} MB)",
                  "ours_ligands_per_s": round(n / (t1 - t0)), "ours_MB_per_s": round(len(text) / 1e6 / (t1 - t0), 1),
                  "threads": os.cpu_count(),
                  "reference_ligands_per_s": round(sample / (t3 - t2)),
                  "reference_sample": f"first {sample} records, single thread (parse_ligand_library)",
                  "speedup": round((n / (t1 - t0)) / (sample / (t3 - t2)), 1)}))
