#!/bin/bash
# A/B timing of the main build against tools/variants/<V> (C2 shape at clash 0.75 / 0.1, C4 shape at 0.1)
# usage: tools/ab.sh OUTDIR [variants...]
out=$1; shift; mkdir -p $out
for c in 0.75 0.1; do
  echo "== main C2 clash $c" >> $out/ab.txt; python tools/prof_run.py --ligands 4000 --runs 3 --clash $c 2>&1 | grep "run 2\|mean best" >> $out/ab.txt
  for v in "$@"; do tools/run_variant.sh $v --ligands 4000 --runs 3 --clash $c 2>&1 | grep "variant\|run 2" >> $out/ab.txt; done
done
echo "== main C4 clash 0.1" >> $out/ab.txt; python tools/prof_run.py --ligands 1000 --atoms 120 --rotamers 32 --runs 3 --clash 0.1 2>&1 | grep "run 2\|mean best" >> $out/ab.txt
for v in "$@"; do tools/run_variant.sh $v --ligands 1000 --atoms 120 --rotamers 32 --runs 3 --clash 0.1 2>&1 | grep "variant\|run 2" >> $out/ab.txt; done
