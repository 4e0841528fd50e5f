"""DRAM traffic per launch of K1a / K1b on a bench workload (ncu counters), -> profiles/traffic_<cfg>.json.

usage (GPU box): python tools/prof_traffic.py c2
Runs ncu on tools/prof_run.py with the config's library size; the JSON is read by bench.py to fill
roofline.traffic (a number measured under ncu is never a bench value; only the byte counts are used).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
sizes = {"c2": ["--ligands", "10000"], "c4": ["--ligands", "1000", "--atoms", "120", "--rotamers", "32"],
         "c5": ["--ligands", "10000", "--dims", "47", "--spacing", "0.375"], "c1": ["--ligands", "100", "--atoms", "32", "--rotamers", "4"]}
metrics = "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum"
cmd = ["ncu", "--metrics", metrics, "--clock-control", "none", "-k", "regex:align_coarse|dock_fast", "--csv",
       sys.executable, os.path.join(ROOT, "tools", "prof_run.py"), "--runs", "1"] + sizes[cfg]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = [r for r in csv.reader(io.StringIO(out[out.index('"ID"'):]))]
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
res = {}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}
for r in rows[1:]:
    k = "k1a" if "align_coarse" in r[ki] else "k1b"
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
    res.setdefault(k, {})[r[mi]] = v
j = {"config": cfg, "source": "ncu --metrics " + metrics + " (one launch each, serialised, cold L2)",
     "k1a_dram_bytes_per_launch": res["k1a"]["dram__bytes_read.sum"] + res["k1a"]["dram__bytes_write.sum"],
     "k1b_dram_bytes_per_launch": res["k1b"]["dram__bytes_read.sum"] + res["k1b"]["dram__bytes_write.sum"],
     "raw": res}
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
json.dump(j, open(os.path.join(ROOT, "profiles", f"traffic_{cfg}.json"), "w"), indent=1)
print(json.dumps(j))
