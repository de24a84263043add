# per-kernel launch list of the n = 1e8 draw stage + one --set full capture of each draw kernel
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none --csv -k regex:k_region -s 4 -c 4 \
   --log-file gpurun_out/p8_launch.csv python scripts/draw_probe.py 1e8 1e9 > /dev/null 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_region -s 4 -c 4 \
   -o gpurun_out/p8_full python scripts/draw_probe.py 1e8 1e9 > gpurun_out/p8_full.log 2>&1; echo ncu_rc=$?
