#!/bin/bash
# tools/build_variant.sh NAME "NVCC_DEFINES" -> tools/variants/NAME/libgeodock_b200.so (experiments only)
set -e
NAME=$1; DEFS=$2
OUT=tools/variants/$NAME; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $DEFS -I include -I paper_1901_06229_b200/csrc -c paper_1901_06229_b200/csrc/gd_fast.cu -o $OUT/gd_fast.cu.o
g++ -shared -o $OUT/libgeodock_b200.so paper_1901_06229_b200/_build/gd_kernels.cu.o $OUT/gd_fast.cu.o paper_1901_06229_b200/_build/gd_capi.cpp.o paper_1901_06229_b200/_build/gd_generate.cpp.o paper_1901_06229_b200/_build/gd_io.cpp.o -L/usr/local/cuda/lib64 -lcudart_static -ldl -lrt -lpthread
