#!/bin/bash
out=gpurun_out/r2e; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.txt
tools/ab.sh $out old
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dock_fast -c 1 -o $out/k1b_c01 python tools/prof_run.py --ligands 2000 --runs 1 --clash 0.1 > $out/ncu_k1b_c01.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dock_fast -c 1 -o $out/k1b_c4_c01 python tools/prof_run.py --ligands 500 --atoms 120 --rotamers 32 --runs 1 --clash 0.1 > $out/ncu_k1b_c4.log 2>&1
