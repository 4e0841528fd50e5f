#!/bin/bash
# swap in the debug build for one run
cp paper_1901_06229_b200/libgeodock_b200.so /tmp/keep.so
cp tools/libgeodock_dbg.so paper_1901_06229_b200/libgeodock_b200.so
python tools/prof_run.py --ligands 300 --runs 1 "$@"
cp /tmp/keep.so paper_1901_06229_b200/libgeodock_b200.so
