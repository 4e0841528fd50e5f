#!/bin/bash
# A/B of the main build against tools/variants/<V>... on the C5 grid (47^3, 0.375 A), 4k ligands
O=gpurun_out/${1:-c5ab}; shift; mkdir -p $O
for c in 0.75 0.1; do
  echo "== main C5 clash $c" >> $O/ab.txt; python tools/prof_run.py --ligands 4000 --dims 47 --spacing 0.375 --runs 3 --clash $c 2>&1 | grep "run 2" >> $O/ab.txt
  for v in "$@"; do tools/run_variant.sh $v --ligands 4000 --dims 47 --spacing 0.375 --runs 3 --clash $c 2>&1 | grep "variant\|run 2" >> $O/ab.txt; done
done
