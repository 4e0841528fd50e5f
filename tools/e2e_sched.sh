O=gpurun_out/r2y; mkdir -p $O
for T in 2 4 16; do for L in 1250 10000; do
  echo "== T=$T L=$L new" >> $O/e2e.txt; GD_HOST_THREADS=$T python tools/e2e_trace.py --ligands $L 2>&1 | grep "e2e ms" | cut -c1-20 >> $O/e2e.txt
  echo "== T=$T L=$L old" >> $O/e2e.txt; GD_CHUNK0=$([ $L -gt 4096 ] && echo 625 || echo 256) GD_CHUNK_GROWTH=4 GD_HOST_THREADS=$T python tools/e2e_trace.py --ligands $L 2>&1 | grep "e2e ms" | cut -c1-20 >> $O/e2e.txt
done; done
