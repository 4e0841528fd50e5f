#!/bin/bash
# tools/run_microbench.sh — build + run the pipe microbenchmarks (on a GPU box)
cd "$(dirname "$0")" && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu && ./microbench
