export GD_PRINT_PHASES=1
for c in 0.75 0.1; do echo "== clash $c"; tools/run_variant.sh phases --ligands 4000 --runs 1 --clash $c 2>&1 | grep -i "phase\|run"; done
