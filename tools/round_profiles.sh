#!/bin/bash
# Round evidence on one B200 (run under gpurun): bench lines, ncu launch list of the bench command,
# full ncu captures of K1a and K1b on the C2 workload, DRAM traffic JSON. Outputs in gpurun_out/.
set -x
O=gpurun_out
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --clash 0.1 --no-cpu > $O/bench_c2_clash01.json 2>> $O/bench_c2.err
python bench.py --config c4 --no-cpu > $O/bench_c4.json 2>> $O/bench_c2.err
python bench.py --config c5 --no-cpu > $O/bench_c5.json 2>> $O/bench_c2.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference_c2.json 2>> $O/bench_c2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu > $O/bench_under_ncu.log 2>&1
python tools/prof_traffic.py c2 > $O/traffic.log 2>&1; cp profiles/traffic_c2.json $O/
for k in align_coarse dock_fast; do
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o $O/ncu_${k}_c2 \
      python tools/prof_run.py --ligands 10000 --runs 1 > /dev/null 2>&1
done
python tools/stream_1m.py > gpurun_out/stream_1m_c5.json 2>> gpurun_out/bench_c2.err
