for v in default minb5 minb6 default; do
  if [ $v = default ]; then L=""; else L=build_variants/$v/libwrs_b200.so; fi
  WRS_B200_LIB=$L timeout 300 python bench.py --no-e2e --no-cpu --steps 10 > gpurun_out/ab_$v.log 2>&1
  echo $v $(tail -1 gpurun_out/ab_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['ms_per_step'],3), round(d['sample']['ms'],3), round(d['aggregate']['ms'],3))")
done
