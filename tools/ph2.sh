export GD_PRINT_PHASES=1
for v in phases phprev; do echo "== $v"; tools/run_variant.sh $v --ligands 4000 --runs 1 --clash 0.1 2>&1 | grep "phase\|run"; done
