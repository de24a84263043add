# GPU suite + builds at the sizes the wave-fit job rule changes
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/jr_tests.log 2>&1; echo tests_rc=$?
for n in 1e7 16777216 1e8 1.25e8 1e9 1073741824; do echo "n=$n $(timeout 300 python scripts/stage_probe.py $n 5 | tail -1)"; done > gpurun_out/jr_stage.log 2>&1
