for c in 0.75 0.1; do echo "== main clash $c"; python tools/prof_run.py --ligands 4000 --runs 3 --clash $c | grep "run 2"; done
echo "== reps0"; python tools/prof_run.py --ligands 4000 --runs 3 --reps 0 | grep "run 2"
