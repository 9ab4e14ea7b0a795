#!/bin/bash
# ncu evidence for the current build (run on the GPU box from the repo root):
#   tools/profile_round.sh <tag>
# plain run first (must exit 0), then: launch list of every libkvring kernel,
# full captures of a decode-step ring-put, a bulk (C5) ring-put and an append.
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CMD="python bench.py --steps 40 --warmup 3 --e2e-steps 0 --nccl-steps 0 --no-cpu-baseline --no-restore --bulk-reps 2"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:kv_ --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
# ring-put launches: 199 prelude + 3 warm-up + 40 timed, then the bulk reps
ncu --set full --clock-control none --import-source on -k regex:kv_ring_put_kernel -s 210 -c 2 \
    -o gpurun_out/ringput_$TAG -f $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:kv_ring_put_kernel -s 243 -c 1 \
    -o gpurun_out/ringput_bulk_$TAG -f $CMD > gpurun_out/ncu_full_bulk_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:kv_append_scatter_kernel -s 210 -c 2 \
    -o gpurun_out/append_$TAG -f $CMD > gpurun_out/ncu_full_append_$TAG.log 2>&1
echo done
