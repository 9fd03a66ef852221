#!/bin/bash
# Build variants/NAME.so: the library with swe.cu recompiled under extra nvcc flags
# (development aid for A/B runs via DC_LIB_PATH; variants/ is git- and not gpurun-ignored). Usage: tools/build_variant.sh NAME [flags...]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
C=$ROOT/paper_1910_01031_b200/csrc
mkdir -p $ROOT/variants/obj_$NAME
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC "$@" -c $C/swe.cu -o $ROOT/variants/obj_$NAME/swe.o
OBJS=$(ls $C/build/*.o | grep -v '/swe.o$')
nvcc $ARCH -shared -o $ROOT/variants/$NAME.so $ROOT/variants/obj_$NAME/swe.o $OBJS
echo built variants/$NAME.so
