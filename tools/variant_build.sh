#!/bin/bash
# Build an experimental libdg variant: recompile ONE translation unit
# (default dg_ops_d3.cu; SRC=dg_vector.cu ... to pick another) with extra
# -D flags, link with the other objects of the current in-tree build.
#   [SRC=dg_vector.cu] tools/variant_build.sh NAME -DFOO=1 ...   ->  _variants/libdg_NAME.so
set -e
NAME=$1; shift
SRC=${SRC:-dg_ops_d3.cu}
OBJ=${SRC%.cu}.o
ROOT=$(cd "$(dirname "$0")/.." && pwd)
B=$ROOT/paper_2408_08129_b200/_build
mkdir -p $ROOT/_variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 \
  -I$ROOT/include -I$ROOT/paper_2408_08129_b200/csrc "$@" \
  -c $ROOT/paper_2408_08129_b200/csrc/$SRC -o $ROOT/_variants/${NAME}_$OBJ
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/_variants/libdg_$NAME.so \
  $(ls $B/*.o | grep -v "/$OBJ") $ROOT/_variants/${NAME}_$OBJ \
  -L/usr/lib/x86_64-linux-gnu -l:libnccl.so.2 -lcudart
echo built _variants/libdg_$NAME.so
