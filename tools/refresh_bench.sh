# bench lines (no ncu) into gpurun_out/; tools/summarize_profiles.sh-style copies are done by hand
O=gpurun_out
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --clash 0.1 --no-cpu > $O/bench_c2_clash01.json 2>> $O/bench_c2.err
python bench.py --config c4 --no-cpu > $O/bench_c4.json 2>> $O/bench_c2.err
python bench.py --config c5 --no-cpu > $O/bench_c5.json 2>> $O/bench_c2.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference_c2.json 2>> $O/bench_c2.err
tail -3 $O/bench_c2.err
