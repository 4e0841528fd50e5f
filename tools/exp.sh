for r in 0 3; do echo "== main reps=$r"; python tools/prof_run.py --ligands 4000 --runs 3 --reps $r | grep "run 2"; done
