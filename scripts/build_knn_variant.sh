#!/bin/bash
# Build ../libcmgpu_<name>.so from the product objects with knn.cu recompiled
# under extra -D flags (kNN A/B variants): build_knn_variant.sh name -DX=1 ...
set -e
cd "$(dirname "$0")/../paper_2502_11602_b200/csrc"
name=$1; shift
mkdir -p ../../build/obj_v_$name
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false -Xptxas -O3,-v \
  -Xcompiler -fPIC,-ffp-contract=off,-O3 -I../../include "$@" -c knn.cu -o ../../build/obj_v_$name/knn.o \
  2> ../../build/obj_v_$name/ptxas.log
objs=$(ls ../../build/obj/*.o | grep -v '/knn.o')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libcmgpu_$name.so $objs ../../build/obj_v_$name/knn.o -lcudart -ldl
grep -A1 "knn_thread_kernelILi2ELi\(8\|16\)ELb0" ../../build/obj_v_$name/ptxas.log | grep "spill\|registers" | head -4
