#!/bin/bash
out=gpurun_out/r2h; mkdir -p $out
tools/ab.sh $out old old_pad inl inl_nofield
for v in old inl; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dock_fast -c 1 -o $out/k1b_075_$v bash tools/run_variant.sh $v --ligands 2000 --runs 1 --clash 0.75 > $out/ncu_075_$v.log 2>&1
done
