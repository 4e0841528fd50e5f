# quick GPU iteration: parity tests, timings at both clash factors, phase split, optional ncu capture
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
export GD_PRINT_PHASES=1
for c in 0.75 0.1; do
  echo "== clash $c"; python tools/prof_run.py --ligands 4000 --runs 3 --clash $c 2>&1 | grep -v "^phase" | grep "run 2"
  [ -d tools/variants/phases ] && tools/run_variant.sh phases --ligands 4000 --runs 1 --clash $c 2>&1 | grep phase
done
if [ -n "$NCU" ]; then
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:dock_fast -c 1 -o gpurun_out/$NCU python tools/prof_run.py --ligands 1500 --runs 1 > /dev/null 2>&1; echo "ncu rc=$?"
fi
