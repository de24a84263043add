# A/B: job length J (WRS_B200_JOB_ITEMS) at several n; wave-filling J = ceil(n / (148*384*w))
mkdir -p gpurun_out
run() { echo "n=$1 J=$2 $(WRS_B200_JOB_ITEMS=$2 timeout 120 python scripts/stage_probe.py $1 5 | tail -1)"; }
{
run 1e8 1024; run 1e8 1760; run 1e8 880; run 1e8 2048; run 1e8 1760; run 1e8 1024
run 1.25e8 1024; run 1.25e8 1100; run 1.25e8 2200
run 1073741824 1024; run 1073741824 1890
run 16777216 256; run 16777216 296
run 1e7 128; run 1e7 176
} > gpurun_out/job_ab.log 2>&1
