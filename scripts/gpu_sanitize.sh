#!/usr/bin/env bash
# compute-sanitizer over the small-n workload (scripts/sanitize_cases.py):
# memcheck, racecheck, synccheck, initcheck.  Summaries go to
# gpurun_out/sanitize_<tool>.txt; the last line of each is the tool's error
# count.  Run on a GPU box:  bash scripts/gpu_sanitize.sh [tools...]
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TOOLS=${*:-memcheck racecheck synccheck initcheck}
CS=/usr/local/cuda/bin/compute-sanitizer
rc=0
for t in $TOOLS; do
  extra=""
  [ "$t" = memcheck ] && extra="--leak-check no"
  timeout 1500 $CS --tool "$t" $extra --print-limit 20 --error-exitcode 9 \
      python scripts/sanitize_cases.py > "gpurun_out/sanitize_$t.txt" 2>&1
  r=$?
  echo "== $t rc=$r" | tee -a "gpurun_out/sanitize_$t.txt"
  tail -3 "gpurun_out/sanitize_$t.txt"
  [ $r -ne 0 ] && rc=$r
done
exit $rc
