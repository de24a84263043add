# region size x tile threads for 1e9 draws at several table sizes (after the bulk unpermute)
mkdir -p gpurun_out
for n in 1e8 268435456 1073741824; do for sh in 20 21 22 23; do for tt in 256 512 1024; do
  echo "n=$n shift=$sh tt=$tt $(WRS_B200_REGION_SHIFT=$sh WRS_B200_TILE_THREADS=$tt timeout 120 python scripts/draw_probe.py $n 1e9 2>&1 | tail -1)"
done; done; done > gpurun_out/region_sweep.log 2>&1
