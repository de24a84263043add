# per-launch device times of one bench step (cold-cache, serialised by ncu):
#   TAG=<name> bash scripts/gpu_launches.sh
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu ${BENCH_ARGS}"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo ncu_rc=$?
python scripts/launch_table.py gpurun_out/launches_${TAG}.csv
