#!/bin/bash
# ncu evidence for the current build (run on the GPU box from the repo root):
#   tools/profile_round.sh <tag>
# plain run first (must exit 0), then: launch list of every libkvring kernel of
# the DEFAULT bench command, and full captures of a decode-step ring-put (inline
# descriptors), a bulk (C5) ring-put and a decode-step append.
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python bench.py > gpurun_out/plain_default_$TAG.log 2>&1 || { echo "plain default run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:kv_ --csv \
    --log-file gpurun_out/launches_default_$TAG.csv python bench.py > gpurun_out/ncu_launch_default_$TAG.log 2>&1
CMD="python bench.py --steps 40 --warmup 3 --e2e-steps 0 --nccl-steps 0 --no-cpu-baseline --no-restore --bulk-reps 2 --interference-steps 0 --block-steps 0 --shared-steps 0"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:kv_ --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
# ring-put launches: 199 prelude (staged kernel) + 3 warm-up + 40 timed (inline kernel), then bulk
ncu --set full --clock-control none --import-source on -k regex:kv_ring_put_copy -s 5 -c 3 \
    -o gpurun_out/ringput_$TAG -f $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:kv_ring_put -s 243 -c 1 \
    -o gpurun_out/ringput_bulk_$TAG -f $CMD > gpurun_out/ncu_full_bulk_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:kv_append_scatter -s 215 -c 2 \
    -o gpurun_out/append_$TAG -f $CMD > gpurun_out/ncu_full_append_$TAG.log 2>&1
for r in ringput ringput_bulk append; do
  ncu -i gpurun_out/${r}_$TAG.ncu-rep --page raw --csv > gpurun_out/${r}_${TAG}_raw.csv 2>/dev/null
  ncu -i gpurun_out/${r}_$TAG.ncu-rep --page details > gpurun_out/${r}_${TAG}_details.txt 2>/dev/null
done
echo done
