#!/bin/bash
out=gpurun_out/r2i; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.txt
tools/ab.sh $out old nohint newrows2
