#!/bin/bash
# variant timing: main library and tools/variants/$V at clash 0.75 / 0.1 (C2 shape, 4000 ligands) and C4 shape at 0.1
out=gpurun_out/r2c; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.txt
for c in 0.75 0.1; do
  echo "== main clash $c" >> $out/exp.txt; python tools/prof_run.py --ligands 4000 --runs 3 --clash $c 2>&1 | grep "run 2" >> $out/exp.txt
  for v in "$@"; do tools/run_variant.sh $v --ligands 4000 --runs 3 --clash $c 2>&1 | grep "variant\|run 2" >> $out/exp.txt; done
done
echo "== main C4 clash 0.1" >> $out/exp.txt; python tools/prof_run.py --ligands 500 --atoms 120 --rotamers 32 --runs 3 --clash 0.1 2>&1 | grep "run 2" >> $out/exp.txt
for v in "$@"; do tools/run_variant.sh $v --ligands 500 --atoms 120 --rotamers 32 --runs 3 --clash 0.1 2>&1 | grep "variant\|run 2" >> $out/exp.txt; done
export GD_PRINT_PHASES=1
tools/run_variant.sh phases --ligands 4000 --runs 2 --clash 0.1 > $out/phases_0.1.txt 2>&1
