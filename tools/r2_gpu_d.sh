#!/bin/bash
# K1a variant A/B (C2) + fresh K1b ncu captures (C2 clash 0.75 / 0.1) of the current main build
O=gpurun_out/${1:-r2d}; shift; mkdir -p $O
for v in "" "$@"; do
  if [ -z "$v" ]; then echo "== main" >> $O/ab.txt; python tools/prof_run.py --ligands 4000 --runs 4 2>&1 | grep "run [23]" >> $O/ab.txt
  else tools/run_variant.sh $v --ligands 4000 --runs 4 2>&1 | grep "variant\|run [23]" >> $O/ab.txt; fi
done
for c in 0.75 0.1; do
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:dock_fast -c 1 -o $O/ncu_k1b_c2_$c \
    python tools/prof_run.py --ligands 10000 --runs 1 --clash $c > $O/ncu_k1b_$c.log 2>&1
done
echo done > $O/DONE
