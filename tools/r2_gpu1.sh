#!/bin/bash
# round-2 GPU session 1: parity suite, FP32 peak, bench lines (N=1, 2 ranks on one GPU, C3 shard), phases
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2/gpu.txt 2>&1
lscpu > gpurun_out/r2/lscpu.txt 2>&1
./tools/fp32_peak > gpurun_out/r2/fp32_peak.json 2> gpurun_out/r2/fp32_peak.err
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2/pytest_gpu.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2/bench_c2.json 2> gpurun_out/r2/bench_c2.err
timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2/bench_c2_n2.json 2> gpurun_out/r2/bench_c2_n2.err
timeout 300 python bench.py --ligands 1250 --steps 5 --no-cpu --no-regimes > gpurun_out/r2/bench_c3_shard8.json 2> gpurun_out/r2/bench_c3_shard8.err
export GD_PRINT_PHASES=1
for c in 0.75 0.1; do
  tools/run_variant.sh phases --ligands 4000 --runs 2 --clash $c > gpurun_out/r2/phases_$c.txt 2>&1
done
unset GD_PRINT_PHASES
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dock_fast -c 1 -o gpurun_out/r2/k1b_c01 python tools/prof_run.py --ligands 2000 --runs 1 --clash 0.1 > gpurun_out/r2/ncu_k1b_c01.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-regimes > gpurun_out/r2/bench_under_ncu.log 2>&1
