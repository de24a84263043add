#!/usr/bin/env bash
# The sanitizer pass of this repo.  compute-sanitizer is closed on the GPU
# pool ("runs under it have left GPUs needing a reset"), so the library checks
# itself: libwrs_b200_checked.so (make -C paper_1903_00227_b200/csrc checked)
# tests every WRS_CHECK'd device index and counts violations, and fills all
# scratch with 0xFF garbage before use (reads of unwritten memory then break
# the parity checks).  scripts/sanitize_cases.py drives every kernel family
# at small n, checks each result against the oracle, and asserts zero
# violations.  Output: gpurun_out/checked.txt.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
[ -f paper_1903_00227_b200/libwrs_b200_checked.so ] || make -s -C paper_1903_00227_b200/csrc checked
WRS_B200_LIB=$PWD/paper_1903_00227_b200/libwrs_b200_checked.so timeout 900 \
    python scripts/sanitize_cases.py > gpurun_out/checked.txt 2>&1
rc=$?
echo "== checked build rc=$rc" | tee -a gpurun_out/checked.txt
tail -4 gpurun_out/checked.txt
exit $rc
