set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "full_size" > gpurun_out/pytest_full.log 2>&1; echo full_rc=$?
python bench.py --steps 3 --warmup 3 --no-e2e > gpurun_out/bench2.log 2>&1; echo bench_rc=$?
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_sample|k_pack|k_partition|k_scan|k_split|k_total" -s 0 -c 8 -o gpurun_out/prof_r1 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
