#!/bin/bash
# round-2 GPU session 2: parity suite, bench (with regimes), phases, ncu of K1b at clash 0.1 and K1a
mkdir -p gpurun_out/r2b
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2b/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b/pytest_gpu.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r2b/bench_c2.json 2> gpurun_out/r2b/bench_c2.err
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2b/bench_c4.json 2> gpurun_out/r2b/bench_c4.err
export GD_PRINT_PHASES=1
for c in 0.75 0.1; do
  tools/run_variant.sh phases --ligands 4000 --runs 2 --clash $c > gpurun_out/r2b/phases_$c.txt 2>&1
done
unset GD_PRINT_PHASES
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dock_fast -c 1 -o gpurun_out/r2b/k1b_c01 python tools/prof_run.py --ligands 2000 --runs 1 --clash 0.1 > gpurun_out/r2b/ncu_k1b_c01.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:align_coarse -c 1 -o gpurun_out/r2b/k1a_c2 python tools/prof_run.py --ligands 4000 --runs 1 > gpurun_out/r2b/ncu_k1a.log 2>&1
