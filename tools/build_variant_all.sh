#!/bin/bash
# Build variants/NAME.so: the whole library recompiled with extra nvcc flags (development
# aid for A/B runs via DC_LIB_PATH). Usage: tools/build_variant_all.sh NAME [flags...]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
SRC=$ROOT/paper_1910_01031_b200/csrc_variant_$NAME
rm -rf $SRC && cp -r $ROOT/paper_1910_01031_b200/csrc $SRC && rm -rf $SRC/build
mkdir -p $ROOT/variants
make -s -C $SRC -j8 NVCC="nvcc $*" OUT=$ROOT/variants/$NAME.so
rm -rf $SRC
echo built variants/$NAME.so
