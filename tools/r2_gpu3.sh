#!/bin/bash
# round-2 GPU session 3 (after the K1b instruction-footprint commits): parity suite, bench lines
# (N=1 with regimes + CPU, 2 ranks on one GPU, C3 shard at N=8, C4), launch list, ncu of K1b at clash 0.1 and K1a
out=gpurun_out/r2d; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/gpu.txt 2>&1
lscpu > $out/lscpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.txt
timeout 900 python bench.py --steps 5 --warmup 3 > $out/bench_c2.json 2> $out/bench_c2.err
timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu > $out/bench_c2_n2.json 2> $out/bench_c2_n2.err
timeout 300 python bench.py --ligands 1250 --steps 5 --no-cpu --no-regimes > $out/bench_c3_shard8.json 2> $out/bench_c3_shard8.err
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > $out/bench_c4.json 2> $out/bench_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-regimes > $out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dock_fast -c 1 -o $out/k1b_c01 python tools/prof_run.py --ligands 2000 --runs 1 --clash 0.1 > $out/ncu_k1b_c01.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:align_coarse -c 1 -o $out/k1a_c2 python tools/prof_run.py --ligands 4000 --runs 1 > $out/ncu_k1a.log 2>&1
for c in 0.75 0.1; do python tools/prof_run.py --ligands 4000 --runs 3 --clash $c > $out/prof_$c.txt 2>&1; done
python tools/prof_run.py --ligands 1000 --atoms 120 --rotamers 32 --runs 3 --clash 0.1 > $out/prof_c4_0.1.txt 2>&1
