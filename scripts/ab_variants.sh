# A/B timing of library variants built by scripts/build_variant.sh (GPU box):
#   VARIANTS="default minb5 ..." bash scripts/ab_variants.sh
# prints: name value ms/step draw-ms aggregate-ms
for v in ${VARIANTS:-default}; do
  case $v in
    default) L="";;
    env:*) L=""; kv=${v#env:}; export ${kv%%,*};;
    *) L=build_variants/$v/libwrs_b200.so;;
  esac
  WRS_B200_LIB=$L timeout 300 python bench.py --no-e2e --no-cpu --steps 10 > gpurun_out/ab_${v//[:=,]/_}.log 2>&1
  echo $v $(tail -1 gpurun_out/ab_${v//[:=,]/_}.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['ms_per_step'],3), round(d['sample']['ms'],3), round(d['aggregate']['ms'],3))")
  case $v in env:*) unset ${kv%%=*};; esac
done
