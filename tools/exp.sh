# per-kernel split (ncu launch list, serialized) for the current build and a variant
for v in main prev; do
  echo "== $v"
  if [ $v = main ]; then cmd="python tools/prof_run.py --ligands 2000 --runs 1"; else cp paper_1901_06229_b200/libgeodock_b200.so /tmp/k.so; cp tools/variants/$v/libgeodock_b200.so paper_1901_06229_b200/; cmd="python tools/prof_run.py --ligands 2000 --runs 1"; fi
  ncu --metrics gpu__time_duration.sum --clock-control none --csv $cmd 2>/dev/null > gpurun_out/launch_$v.csv
  python tools/prof_run.py --ligands 2000 --runs 1 | grep mean
  if [ $v != main ]; then cp /tmp/k.so paper_1901_06229_b200/libgeodock_b200.so; fi
done
