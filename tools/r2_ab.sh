#!/bin/bash
# GPU tests of the current build, then A/B timing of the main build against tools/variants/<V>...
# usage: tools/r2_ab.sh OUTNAME [variants...]
O=gpurun_out/$1; shift; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
tools/ab.sh $O "$@"
echo done > $O/DONE
