#!/usr/bin/env bash
# Build a variant of the library with extra compile flags for A/B timing:
#   bash scripts/build_variant.sh NAME "-DK4_WARPS_DEF=11 ..."
# -> build_variants/NAME/libwrs_b200.so (select with WRS_B200_LIB=...)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
make -s -j8 -C paper_1903_00227_b200/csrc OUT=$PWD/build_variants/$name/libwrs_b200.so \
    BUILD=$PWD/build_variants/$name/obj EXTRA="$*" all
