# quick GPU cycle: parity tests + smoke + bench (no ncu)
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo bench_rc=$?
tail -c 3000 gpurun_out/bench.log
