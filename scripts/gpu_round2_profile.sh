# Round-2 evidence on the GPU box (run under gpurun, each ncu pass only after
# its plain run exited 0):
#   TAG=r02 bash scripts/gpu_round2_profile.sh
# bench line (driver defaults), the ncu launch list of one bench step, and one
# --set full capture of every kernel of the step.
TAG=${TAG:-r02}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_${TAG}.log 2> gpurun_out/bench_${TAG}.err; echo bench_rc=$?
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-aggregate --no-config2"
timeout 600 $CMD > gpurun_out/plain_${TAG}.log 2>&1; echo plain_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo ncu1_rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on \
    -k regex:"k_region|k_pack|k_assemble|k_partition|k_scan|k_split|k_totals|k_carry|k_ckpt" -s 0 -c 19 \
    -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1; echo ncu2_rc=$?
