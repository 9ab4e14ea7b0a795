#!/bin/bash
# ncu evidence for the bench's step kernel (gpurun, ONE GPU), from the repo root:
#   tools/profile_bench.sh <tag>
# 1. the driver's command runs plain (must exit 0);
# 2. launch list of the same command: every kv_step_kernel launch of the prelude (399),
#    warm-up (5) and timed region (20) with its device time and DRAM bytes (cold-cache,
#    serialised: compare SHARES, not absolutes);
# 3. one --set full capture of 3 timed-region launches (traffic per launch).
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
CMD="python bench.py --steps 20 --warmup 5"
$CMD > gpurun_out/${TAG}_plain.jsonl 2> gpurun_out/${TAG}_plain.err || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:kv_step_kernel -c 424 --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:kv_step_kernel -s 409 -c 3 \
    -o gpurun_out/${TAG}_step -f $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
ncu -i gpurun_out/${TAG}_step.ncu-rep --page raw --csv > gpurun_out/${TAG}_step_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_step.ncu-rep --page details > gpurun_out/${TAG}_step_details.txt 2>/dev/null
echo done
