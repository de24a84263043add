# Round evidence on the GPU box (run under gpurun):
#   TAG=r01 bash scripts/gpu_round1_profile.sh
# full parity suite, the default bench line, then (each after its plain run
# exited 0) the ncu launch list of one bench step and one --set full capture
# of every kernel of the step.
set -x
TAG=${TAG:-r01}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_all_${TAG}.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_all_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.log 2>&1; echo bench_rc=$?
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_${TAG}.log 2>&1; echo plain_rc=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo ncu1_rc=$?
ncu --set full --clock-control none --import-source on \
    -k regex:"k_region|k_pack|k_assemble|k_partition|k_scan|k_split" -s 0 -c 19 \
    -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1; echo ncu2_rc=$?
