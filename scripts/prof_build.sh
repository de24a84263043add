# ncu --set full of the build kernels at n=1e8 (one rebuild after the first
# build), e.g.  KREGEX='k_pack|k_assemble' bash scripts/prof_build.sh tag
TAG=${1:-x}
KREGEX=${KREGEX:-k_pack|k_assemble|k_partition|k_scan|k_split}
mkdir -p gpurun_out
python scripts/stage_probe.py 1e8 5 > gpurun_out/stages_${TAG}.txt 2>&1; echo plain_rc=$?
cat gpurun_out/stages_${TAG}.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" \
    -s ${SKIP:-2} -c ${COUNT:-2} -o gpurun_out/prof_${TAG} python scripts/stage_probe.py 1e8 1 \
    > gpurun_out/ncu_${TAG}.log 2>&1; echo ncu_rc=$?
