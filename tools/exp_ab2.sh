# tools/exp_ab2.sh V : main vs variant V on C2 (clash 0.75 / 0.1) and C4 (clash 0.1)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for i in 1 2; do for a in "--clash 0.75" "--clash 0.1" "--ligands 1000 --atoms 120 --rotamers 32 --clash 0.1"; do
  echo "== $a"; python tools/prof_run.py --ligands 4000 --runs 3 $a | grep "run 2"; tools/run_variant.sh $1 --ligands 4000 --runs 3 $a | grep "run 2"
done; done
