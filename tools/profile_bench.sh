#!/bin/bash
# Usage (on the GPU box, from the repo root): tools/profile_bench.sh <tag>
# Plain run first (must exit 0), then the ncu launch list and one full capture
# of the ring-put kernel in the timed region.  Outputs under gpurun_out/.
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
CMD="python bench.py --steps 40 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:kv_ --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:kv_ring_put_kernel -s 215 -c 3 \
    -o gpurun_out/ringput_$TAG -f $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:kv_append_scatter_kernel -s 215 -c 2 \
    -o gpurun_out/append_$TAG -f $CMD > gpurun_out/ncu_full_append_$TAG.log 2>&1
echo done
