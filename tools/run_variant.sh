#!/bin/bash
# tools/run_variant.sh NAME args... : run tools/prof_run.py with a variant library swapped in
NAME=$1; shift
cp paper_1901_06229_b200/libgeodock_b200.so /tmp/keep_main.so
cp tools/variants/$NAME/libgeodock_b200.so paper_1901_06229_b200/libgeodock_b200.so
echo "== variant $NAME"; python tools/prof_run.py "$@"
cp /tmp/keep_main.so paper_1901_06229_b200/libgeodock_b200.so
