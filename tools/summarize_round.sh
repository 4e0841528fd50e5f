#!/bin/bash
# Turn gpurun_out/<dir> (from tools/r2_round.sh) into the tracked summaries under profiles/<round>_*.
# usage: tools/summarize_round.sh gpurun_out/r2a r2

D=$1; R=$2
for f in bench_c2 bench_c4 bench_c5 bench_c1 bench_reference_c2; do
  [ -f $D/$f.json ] && tail -n 1 $D/$f.json > profiles/${R}_$f.json
done
[ -f $D/traffic_c2.json ] && cp $D/traffic_c2.json profiles/traffic_c2.json
python3 - "$D" <<'PY' > profiles/${R}_launches_c2.txt
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1] + '/launches_c2.csv')))
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
summ() {  # report title out
  ncu -i $1 --page source --csv --print-source=cuda,sass > /tmp/_s.csv 2>/dev/null
  (echo "# $2"; tools/ncu_summary.sh $1; echo; echo "# hottest source lines"; python3 tools/ncu_lines.py /tmp/_s.csv 25 2>/dev/null
   if [ -n "$4" ]; then echo; echo "# per-phase (SASS attributed to kernel-body regions)"; python3 tools/ncu_phases.py /tmp/_s.csv 2>/dev/null; fi) > $3
}
[ -f $D/ncu_k1a_c2.ncu-rep ] && summ $D/ncu_k1a_c2.ncu-rep "ncu --set full, K1a align_coarse_kernel, C2 10k ligands (tools/prof_run.py --ligands 10000)" profiles/${R}_ncu_k1a_c2_summary.txt
[ -f $D/ncu_k1b_c2_0.75.ncu-rep ] && summ $D/ncu_k1b_c2_0.75.ncu-rep "ncu --set full, K1b dock_fast_kernel, C2 10k ligands, clash 0.75 (default)" profiles/${R}_ncu_k1b_c2_summary.txt phases
[ -f $D/ncu_k1b_c2_0.1.ncu-rep ] && summ $D/ncu_k1b_c2_0.1.ncu-rep "ncu --set full, K1b dock_fast_kernel, C2 10k ligands, clash 0.1 (commit path live)" profiles/${R}_ncu_k1b_c2_clash01_summary.txt phases
echo done
