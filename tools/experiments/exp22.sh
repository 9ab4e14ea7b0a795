# fused loop (1 launch / step) with whole-item tasks (128 segs = 32 KiB: one load round per CTA)
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
B="bench.py --no-cpu-baseline --e2e-steps 0 --no-restore --nccl-steps 0 --bulk-reps 0 --interference-steps 0 --block-steps 0 --shared-steps 0 --steps 400"
for r in 1 2; do
for v in "X=1 --loop streams" "X=1 --loop fused" "KVRING_MIN_TASK_SEGS=128 --loop fused" "KVRING_MIN_TASK_SEGS=128 --loop pdl" "X=1 --loop pdl"; do
  set -- $v
  echo "== $v round $r" >> gpurun_out/exp22.log
  env $1 timeout 300 python $B $2 $3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['kernel_us']['median'], d['roofline']['frac'], d['clocks']['sm_mhz'], {k: d['host_us_per_step'][k] for k in ('prepare','wait_prepare','stage_h2d','stage.acquire_wait','launch_append','launch_publish')})" >> gpurun_out/exp22.log 2>&1
done; done
