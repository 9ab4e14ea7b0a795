# append grid cap (the ring-put of step k runs concurrently with the append of k+1)
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
B="bench.py --no-cpu-baseline --e2e-steps 0 --no-restore --nccl-steps 0 --bulk-reps 0 --interference-steps 0 --block-steps 0 --shared-steps 0 --steps 400"
for r in 1 2; do
for v in "X=1" "KVRING_APPEND_CTAS_PER_SM=1" "KVRING_APPEND_CTAS_PER_SM=2"; do
  echo "== $v round $r" >> gpurun_out/exp25.log
  env $v timeout 300 python $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); h=d['host_us_per_step']; print(d['value'], d['ms_per_step'], d['kernel_us']['median'], d['kernel_us']['avg'], {k: h[k] for k in ('stage.acquire_wait','launch_publish','worker_wait_issue')})" >> gpurun_out/exp25.log 2>&1
done; done
