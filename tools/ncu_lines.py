"""Aggregate an ncu source page (--print-source=cuda,sass --csv) per CUDA source line.

usage: ncu -i X.ncu-rep --page source --csv --print-source=cuda,sass > s.csv; python tools/ncu_lines.py s.csv
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
out, fname, cur = [], None, None
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr is None or len(r) < 5:
        continue
    if r[0] not in ("", None) and r[0].isdigit():
        try:
            samples = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
            iv = r[hdr["Instructions Executed"]]
            instr = float(iv) if iv not in ("", "-") else 0.0
        except (ValueError, IndexError):
            continue
        out.append((samples, instr, f"{fname}:{r[0]}", r[1][:90]))
tot_s = sum(o[0] for o in out) or 1
tot_i = sum(o[1] for o in out) or 1
print(f"total samples {tot_s:.0f}  total warp-instr {tot_i:.3e}")
for s, i, where, src in sorted(out, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 45]:
    print(f"{100 * s / tot_s:5.1f}% smp {100 * i / tot_i:5.1f}% ins  {where:18s} {src}")
