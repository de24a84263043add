# tile threads (unpermute tile = TT * 16 draws) with the 32-row scatter, and counts A/B
mkdir -p gpurun_out
for n in 2e7 5e7 1e8 268435456 1073741824; do for tt in 256 512 1024; do
  echo "n=$n tt=$tt $(WRS_B200_TILE_THREADS=$tt timeout 120 python scripts/draw_probe.py $n 1e9 | tail -1)"; done; done > gpurun_out/ttr.log 2>&1
for r in 16 32; do echo "counts rows=$r $(WRS_B200_SCATTER_ROWS=$r timeout 300 python bench.py --no-e2e --no-cpu --no-config2 --steps 3 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["aggregate"]["ms"], d["sample"]["ms"], d["ms_per_step"])')"; done >> gpurun_out/ttr.log 2>&1
