for i in 1 2; do for a in "--clash 0.75" "--clash 0.1"; do
  echo "== C4 $a"; python tools/prof_run.py --ligands 1000 --atoms 120 --rotamers 32 --runs 3 $a | grep "run 2"
  for v in n4t384 n4t256; do tools/run_variant.sh $v --ligands 1000 --atoms 120 --rotamers 32 --runs 3 $a | grep "run 2"; done
done; done
