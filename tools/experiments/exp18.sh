# two-stream loop with inline (parameter-space) descriptors vs staged descriptors
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/exp18_tests.log 2>&1
B="bench.py --no-cpu-baseline --e2e-steps 0 --no-restore --nccl-steps 0 --bulk-reps 0 --interference-steps 0 --block-steps 0 --shared-steps 0 --steps 400"
for v in "X=1 --loop streams" "KVRING_MIN_TASK_SEGS=128 --loop streams" "X=1 --loop pdl" "X=1 --loop streams" "KVRING_MIN_TASK_SEGS=128 --loop streams"; do
  set -- $v
  echo "== $v" >> gpurun_out/exp18.log
  env $1 timeout 300 python $B $2 $3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['kernel_us'], d['roofline']['frac']); print(d['host_us_per_step'])" >> gpurun_out/exp18.log 2>&1
done
