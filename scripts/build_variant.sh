#!/bin/bash
# build libgacer.so variants with extra nvcc defines into ab_libs/NAME.so
# usage: scripts/build_variant.sh NAME "-DGACER_EPI_V=1 ..."
set -e
NAME=$1; shift
DEFS="$*"
mkdir -p ab_libs /tmp/abv_$NAME
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $DEFS"
C=paper_2304_11745_b200/csrc
nvcc $F -Xptxas=-O3 -c $C/executor.cu -o /tmp/abv_$NAME/executor.o
nvcc $F -Xptxas=-O3 -c $C/train_ops.cu -o /tmp/abv_$NAME/train_ops.o
nvcc $F -c $C/host.cpp -o /tmp/abv_$NAME/host.o
nvcc -shared $F /tmp/abv_$NAME/*.o -o ab_libs/$NAME.so -lcudart
echo built ab_libs/$NAME.so
