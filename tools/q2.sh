timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for i in 1 2; do
echo "== main"; for a in "" "--dims 47 --spacing 0.375" "--clash 0.1" "--ligands 1000 --atoms 120 --rotamers 32"; do python tools/prof_run.py --ligands 4000 --runs 3 $a | grep "run 2"; done
echo "== k1bord"; for a in "" "--dims 47 --spacing 0.375" "--clash 0.1" "--ligands 1000 --atoms 120 --rotamers 32"; do tools/run_variant.sh k1bord --ligands 4000 --runs 3 $a | grep "run 2"; done
done
