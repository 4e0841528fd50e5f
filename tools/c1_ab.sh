#!/bin/bash
# A/B of the main build against tools/variants/<V>... on the C1 shape (32 atoms, 4 rotamers: NS = 1), 4k ligands
O=gpurun_out/${1:-c1ab}; shift; mkdir -p $O
echo "== main C1 shape" >> $O/ab.txt; python tools/prof_run.py --ligands 4000 --atoms 32 --rotamers 4 --runs 3 2>&1 | grep "run 2" >> $O/ab.txt
for v in "$@"; do tools/run_variant.sh $v --ligands 4000 --atoms 32 --rotamers 4 --runs 3 2>&1 | grep "variant\|run 2" >> $O/ab.txt; done
