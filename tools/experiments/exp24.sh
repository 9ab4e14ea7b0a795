# issue-thread breakdown: publication staging vs launch; inline vs staged launch counts
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
B="bench.py --no-cpu-baseline --e2e-steps 0 --no-restore --nccl-steps 0 --bulk-reps 0 --interference-steps 0 --block-steps 0 --shared-steps 0 --steps 400"
for v in "X=1" "KVRING_MIN_TASK_SEGS=128"; do
  echo "== $v" >> gpurun_out/exp24.log
  env $v timeout 300 python $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['kernel_us']['median']); print(d['host_us_per_step'])" >> gpurun_out/exp24.log 2>&1
done
