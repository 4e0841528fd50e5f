#!/bin/bash
# Round-2 call B: GPU tests after the packer rewrite, host packing at 8-GPU concurrency on the box's
# cores, the C3 shard tail (1,250 ligands on one GPU), two and four ranks sharing the GPU (gloo),
# compute-sanitizer on the current kernels.
O=gpurun_out/${1:-r2b}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python tools/host_pack_scale.py > $O/host_pack.json 2> $O/host_pack.err
timeout 600 python bench.py --ligands 1250 --no-cpu > $O/bench_c2_1250.json 2> $O/bench.err
timeout 900 python bench.py --gpus 2 --no-cpu > $O/bench_c2_gpus2.json 2>> $O/bench.err
timeout 900 python bench.py --gpus 4 --no-cpu --no-regimes > $O/bench_c2_gpus4.json 2>> $O/bench.err
lscpu > $O/lscpu.txt 2>&1
timeout 300 python tools/bench_ingest.py 100000 > $O/ingest.json 2> $O/ingest.err
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t python tools/sanitize_case.py > $O/sanitizer_$t.txt 2>&1
done
echo done > $O/DONE
