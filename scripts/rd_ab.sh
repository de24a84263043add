# A/B: unpermute run staging (bulk vs LDGSTS) at n = 1e8 and 2^30, then the region tests
mkdir -p gpurun_out
for rd in 1 0 1 0; do
  echo "rd=$rd $(WRS_B200_RD_BULK=$rd timeout 120 python scripts/draw_probe.py 1e8 1e9 | tail -1)"
  echo "rd=$rd $(WRS_B200_RD_BULK=$rd timeout 120 python scripts/draw_probe.py 1073741824 1e9 | tail -1)"
done > gpurun_out/rd_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "region or golden or draws" > gpurun_out/rd_tests.log 2>&1; echo tests_rc=$?
