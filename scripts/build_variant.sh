#!/bin/bash
# A/B builds of libwrs_b200.so with extra nvcc defines, for timing experiments:
#   bash scripts/build_variant.sh NAME -DFOO=1 ...  -> build_variants/NAME/libwrs_b200.so
# then WRS_B200_LIB=build_variants/NAME/libwrs_b200.so python bench.py ...
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
D=$ROOT/build_variants/$NAME
mkdir -p "$D"
make -s -C "$ROOT/paper_1903_00227_b200/csrc" BUILD="$D/obj" OUT="$D/libwrs_b200.so" NVCC="nvcc $*" -j4
