# ncu capture of selected kernels on the GPU box (run under gpurun):
#   KREGEX=<kernel regex> COUNT=<launches> TAG=<report name> bash scripts/gpu_ncu.sh
# The same command runs plain first and must exit 0 before ncu touches it.
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu ${BENCH_ARGS}"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:${KREGEX}" -c ${COUNT:-8} \
    -o gpurun_out/${TAG} $CMD > gpurun_out/ncu_${TAG}.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/ncu_${TAG}.log
