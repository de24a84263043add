# A/B of a library variant on the draw stage (n = 1e8 and 2^30): default vs build_variants/$V
mkdir -p gpurun_out
for rep in 1 2; do for v in default ${V:-late}; do for n in 1e8 1073741824; do
  L=""; [ $v != default ] && L=$PWD/build_variants/$v/libwrs_b200.so
  echo "$v n=$n $(WRS_B200_LIB=$L python scripts/draw_probe.py $n 1e9 | tail -1)"
done; done; done > gpurun_out/gab.log 2>&1
