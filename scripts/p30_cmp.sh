# per-kernel time / DRAM bytes at n = 2^30 for 32-MB (shift 21) vs 64-MB (22) regions
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for cfg in "21 1024" "21 512" "22 512"; do set -- $cfg
 WRS_B200_REGION_SHIFT=$1 WRS_B200_TILE_THREADS=$2 timeout 600 ncu --metrics $M --clock-control none --csv -k regex:k_region -s 4 -c 4 \
   --log-file gpurun_out/p30c_$1_$2.csv python scripts/draw_probe.py 1073741824 1e9 > /dev/null 2>&1; echo rc=$?
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_region_unpermute -s 1 -c 1 \
   -o gpurun_out/p30_unperm python scripts/draw_probe.py 1073741824 1e9 > gpurun_out/p30_unperm.log 2>&1; echo ncu_rc=$?
