# bench lines + 1M stream (no ncu): tracked copies go to profiles/ via tools/summarize_profiles.sh-style copies
O=gpurun_out
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --clash 0.1 --no-cpu > $O/bench_c2_clash01.json 2>> $O/bench_c2.err
python bench.py --config c4 --no-cpu > $O/bench_c4.json 2>> $O/bench_c2.err
python bench.py --config c5 --no-cpu > $O/bench_c5.json 2>> $O/bench_c2.err
python tools/stream_1m.py > $O/stream_1m_c5.json 2>> $O/bench_c2.err
tail -3 $O/bench_c2.err
