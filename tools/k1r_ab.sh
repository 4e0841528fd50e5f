O=gpurun_out/${1:-k1rab}; mkdir -p $O
for v in main r640 r768 r1024; do
  if [ $v = main ]; then python tools/prof_run.py --ligands 10000 --runs 3 2>&1 | grep "run 2" | sed "s/^/main /" >> $O/ab.txt
  else tools/run_variant.sh $v --ligands 10000 --runs 3 2>&1 | grep "run 2" | sed "s/^/$v /" >> $O/ab.txt; fi
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:align_refine --csv python tools/prof_run.py --ligands 10000 --runs 1 > $O/k1r_main.csv 2>/dev/null
for v in r640 r768 r1024; do cp paper_1901_06229_b200/libgeodock_b200.so /tmp/keep.so; cp tools/variants/$v/libgeodock_b200.so paper_1901_06229_b200/; timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:align_refine --csv python tools/prof_run.py --ligands 10000 --runs 1 > $O/k1r_$v.csv 2>/dev/null; cp /tmp/keep.so paper_1901_06229_b200/libgeodock_b200.so; done
