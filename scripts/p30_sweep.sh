# n = 2^30 draw-stage knobs (region size, tile threads) + one --set full capture
mkdir -p gpurun_out
for sh in 21 22 23; do for tt in 256 512 1024; do
  echo "shift=$sh tt=$tt $(WRS_B200_REGION_SHIFT=$sh WRS_B200_TILE_THREADS=$tt timeout 120 python scripts/draw_probe.py 1073741824 1e9 2>&1 | tail -1)"
done; done > gpurun_out/p30_sweep.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_region -s 4 -c 3 \
   -o gpurun_out/p30_full python scripts/draw_probe.py 1073741824 1e9 > gpurun_out/p30_full.log 2>&1; echo ncu_rc=$?
