# tools/exp_variants.sh V1 V2 ... : main library and each tools/variants/V at both clash factors
for c in 0.75 0.1; do
  echo "== main clash $c"; python tools/prof_run.py --ligands 4000 --runs 3 --clash $c | grep "run 2"
  for v in "$@"; do tools/run_variant.sh $v --ligands 4000 --runs 3 --clash $c | grep "variant\|run 2"; done
done
