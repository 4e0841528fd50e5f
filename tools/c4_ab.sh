#!/bin/bash
# A/B of the main build against tools/variants/<V>... on the C4 shape (1k x 120 atoms x 32 rotamers)
O=gpurun_out/${1:-c4ab}; shift; mkdir -p $O
for c in 0.75 0.1; do
  echo "== main C4 clash $c" >> $O/ab.txt; python tools/prof_run.py --ligands 1000 --atoms 120 --rotamers 32 --runs 3 --clash $c 2>&1 | grep "run 2" >> $O/ab.txt
  for v in "$@"; do tools/run_variant.sh $v --ligands 1000 --atoms 120 --rotamers 32 --runs 3 --clash $c 2>&1 | grep "variant\|run 2" >> $O/ab.txt; done
done
