#!/bin/bash
# Build ../libcmgpu_<name>.so from the product objects with ONE .cu recompiled
# under extra -D flags (A/B variants): build_cu_variant.sh name file.cu -DX=1 ...
set -e
cd "$(dirname "$0")/../paper_2502_11602_b200/csrc"
name=$1; src=$2; shift 2
stem=${src%.cu}
mkdir -p ../../build/obj_v_$name
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false -Xptxas -O3,-v \
  -Xcompiler -fPIC,-ffp-contract=off,-O3 -I../../include "$@" -c $src -o ../../build/obj_v_$name/$stem.o \
  2> ../../build/obj_v_$name/ptxas.log
objs=$(ls ../../build/obj/*.o | grep -v "/$stem.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libcmgpu_$name.so $objs ../../build/obj_v_$name/$stem.o -lcudart -ldl
