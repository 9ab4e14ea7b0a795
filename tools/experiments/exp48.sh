# slot high-water mark loops in prepare; full GPU suite + bench x3
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/exp48_tests.log 2>&1
B="bench.py --no-cpu-baseline --e2e-steps 0 --no-restore --nccl-steps 0 --bulk-reps 0 --interference-steps 0 --block-steps 0 --shared-steps 0 --steps 400"
for r in 1 2 3; do
  timeout 300 python $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); h=d['host_us_per_step']; print(d['value'], d['ms_per_step'], d['kernel_us']['median'], d['kernel_us']['avg'], {k: h[k] for k in ('prepare','prepare.append','prepare.replicate','wait_prepare','worker_wait_issue','stage.acquire_wait')})" >> gpurun_out/exp48.log 2>&1
done
