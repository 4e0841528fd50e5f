#!/bin/bash
out=gpurun_out/r2m; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.txt
tools/ab.sh $out prev
GD_NO_TWINS=1 python tools/prof_run.py --ligands 4000 --runs 3 > $out/notwins.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:align_coarse -c 1 -o $out/k1a_c2 python tools/prof_run.py --ligands 4000 --runs 1 > $out/ncu_k1a.log 2>&1
