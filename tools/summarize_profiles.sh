#!/bin/bash
# Turn gpurun_out/ (from tools/round_profiles.sh) into the tracked summaries under profiles/.
set -e
R=${1:-r1}
for f in bench_c2 bench_c2_clash01 bench_c4 bench_c5 bench_reference_c2; do cp gpurun_out/$f.json profiles/${R}_$f.json; done
cp gpurun_out/traffic_c2.json profiles/traffic_c2.json
python3 - "$R" <<'PY' > profiles/${1:-r1}_launches_c2.txt
import csv, collections, sys
rows = list(csv.reader(open('gpurun_out/launches_c2.csv')))
h = [r for r in rows if r and r[0] == 'ID'][0]
ki, vi = h.index('Kernel Name'), h.index('Metric Value')
tot = collections.OrderedDict(); cnt = collections.Counter()
for r in rows:
    if len(r) > vi and r[0].isdigit():
        name = r[ki].split('(')[0]
        tot[name] = tot.get(name, 0) + float(r[vi].replace(',', '')); cnt[name] += 1
s = sum(tot.values())
print("ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py --steps 2 --warmup 1 --no-cpu")
print("(per-launch times are serialised and cold-cache under ncu; compare shares, not absolutes)\n")
print(f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda t: -t[1]):
    print(f"{k[:60]:60s} {cnt[k]:8d} {v/1e6:10.3f} {100*v/s:6.1f}%")
PY
ncu -i gpurun_out/ncu_align_coarse_c2.ncu-rep --page source --csv --print-source=cuda,sass > /tmp/_a.csv 2>/dev/null
ncu -i gpurun_out/ncu_dock_fast_c2.ncu-rep --page source --csv --print-source=cuda,sass > /tmp/_b.csv 2>/dev/null
(echo "# ncu --set full, K1a align_coarse_kernel<2,512,true>, C2 10k ligands (tools/prof_run.py --ligands 10000)"
 tools/ncu_summary.sh gpurun_out/ncu_align_coarse_c2.ncu-rep; echo; echo "# hottest source lines"
 python tools/ncu_lines.py /tmp/_a.csv 25 2>/dev/null) > profiles/${R}_ncu_k1a_c2_summary.txt
(echo "# ncu --set full, K1b dock_fast_kernel<2,512,*>, C2 10k ligands"
 tools/ncu_summary.sh gpurun_out/ncu_dock_fast_c2.ncu-rep; echo; echo "# per-phase (SASS attributed to kernel-body regions)"
 python tools/ncu_phases.py /tmp/_b.csv) > profiles/${R}_ncu_k1b_c2_summary.txt
echo done
