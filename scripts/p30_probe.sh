mkdir -p gpurun_out
python scripts/draw_probe.py 1073741824 1e9 > gpurun_out/p30_plain.log 2>&1; echo rc=$?
python scripts/draw_probe.py 1e9 2147483648 >> gpurun_out/p30_plain.log 2>&1; echo rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none --csv -k regex:k_region --log-file gpurun_out/p30_launches.csv python scripts/draw_probe.py 1073741824 1e9 > gpurun_out/p30_ncu.log 2>&1; echo ncu_rc=$?
