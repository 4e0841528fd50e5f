#!/bin/bash
# Round-2 evidence on one B200 (run under gpurun): GPU tests, smoke, bench lines, launch list,
# ncu --set full of K1a and of K1b at clash 0.75 and 0.1, DRAM traffic. Outputs in gpurun_out/$1.
O=gpurun_out/${1:-r2}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
nvidia-smi -q -d CLOCK,PERFORMANCE > $O/clocks_before.txt 2>&1
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench.err
timeout 600 python bench.py --config c4 --no-cpu > $O/bench_c4.json 2>> $O/bench.err
timeout 600 python bench.py --config c5 --no-cpu > $O/bench_c5.json 2>> $O/bench.err
timeout 600 python bench.py --config c1 --no-cpu > $O/bench_c1.json 2>> $O/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference_c2.json 2>> $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu > $O/bench_under_ncu.log 2>&1
timeout 600 python tools/prof_traffic.py c2 > $O/traffic.log 2>&1; cp profiles/traffic_c2.json $O/
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:align_coarse -c 1 -o $O/ncu_k1a_c2 \
    python tools/prof_run.py --ligands 10000 --runs 1 > $O/ncu_k1a.log 2>&1
for c in 0.75 0.1; do
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:dock_fast -c 1 -o $O/ncu_k1b_c2_$c \
    python tools/prof_run.py --ligands 10000 --runs 1 --clash $c > $O/ncu_k1b_$c.log 2>&1
done
echo done > $O/DONE
