#!/bin/bash
out=gpurun_out/${1:-r2n}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.txt
tools/ab.sh $out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv python tools/prof_run.py --ligands 4000 --runs 2 --clash 0.1 > $out/launches.log 2>&1
for c in 0.75 0.1; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dock_fast -c 1 -o $out/k1b_$c python tools/prof_run.py --ligands 2000 --runs 1 --clash $c > $out/ncu_k1b_$c.log 2>&1
done
