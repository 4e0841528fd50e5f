"""Per-phase (source-region) breakdown of an ncu source page for dock_fast_kernel.

usage: ncu -i X --page source --csv --print-source=cuda,sass > s.csv; python tools/ncu_phases.py s.csv
Inlined helper lines are attributed to the phase of the call site by SASS address order: every
SASS instruction belongs to the last gd_fast.cu kernel-body line seen before it.
"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
src = open(__file__.replace("tools/ncu_phases.py", "paper_1901_06229_b200/csrc/gd_fast.cu")).read().split("\n")


def find(pat):
    lines = pat.split("\n")
    for i in range(len(src)):
        if all(lines[k].strip() in src[i + k] for k in range(len(lines)) if i + k < len(src)):
            return i + 1
    raise KeyError(pat)


marks = [("setup/aligned-pose", find("dock_fast_kernel(DevPocket pk")),
         ("sweep-setup+refresh", find("dihedral sweep (docking.cpp:155-167")),
         ("step-head", find("for (uint32_t rep = 0; rep < pr.reps; ++rep)")),
         ("step-axis", find("coarse evaluation of every candidate k = 1")),
         ("step-pairs", find("Cross pairs (DESIGN.md §3.2). Rotating M' by theta")),
         ("step-cand-setup", find("const uint32_t n_cand = pr.S - 1;  // k = 1 .. S-1")),
         ("step-cand-loop", find("for (uint32_t mq = s0 + 1 + sub; mq < e0; mq += gs) {")),
         ("step-cand-reduce", find("for (uint32_t o = 1; o < gs; o <<= 1) {  // group reduction")),
         ("step-decisions", find("exact decisions (reference semantics")),
         ("step-commit", find("commit = rotate_fragment(current, r, k*delta)")),
         ("restart-tail", find("restart result"))]
kstart = marks[0][1]
# prologue lines (lane, smem bases, grid constants) are rematerialised inside loops: transparent
kloop = next(i + 1 for i in range(kstart, len(src)) if src[i].strip().startswith("for (;;) {"))
# pass 1: collect (address, instr, samples, (file, line)) in page order
hdr, fname, cur = None, None, None
ins_rows = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr is None or len(r) < 6:
        continue
    if r[0].isdigit():
        cur = (fname, int(r[0]))
        continue
    if r[0] == "" and r[2].startswith("0x"):
        try:
            ins = float(r[hdr["Instructions Executed"]] or 0)
            smp = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        ins_rows.append((int(r[2], 16), ins, smp, cur))
ins_rows.sort()
phase, agg = "k1b-prologue", {}
for addr, ins, smp, (f, l) in ins_rows:
    if f == "gd_fast.cu" and l > kloop:
        phase = [m for m, ln in marks if ln <= l][-1]
    a = agg.setdefault(phase, [0.0, 0.0])
    a[0] += ins
    a[1] += smp
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"{'phase':24s} {'instr %':>8s} {'samples %':>10s}")
for k, (i, s) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:24s} {100 * i / ti:8.1f} {100 * s / ts:10.1f}")
