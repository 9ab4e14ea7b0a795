# CUDA-graph decode loop: parity tests, then interleaved A/B vs the two-stream loop
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "graph or run_steps" > gpurun_out/exp34_tests.log 2>&1 || exit 1
B="bench.py --no-cpu-baseline --e2e-steps 0 --no-restore --nccl-steps 0 --bulk-reps 0 --interference-steps 0 --block-steps 0 --shared-steps 0 --steps 400"
for r in 1 2; do
for v in streams graph; do
  echo "== $v round $r" >> gpurun_out/exp34.log
  timeout 300 python $B --loop $v 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); h=d['host_us_per_step']; print(d['value'], d['ms_per_step'], d['kernel_us']['median'], d['kernel_us']['avg'], d['roofline']['frac'], {k: h[k] for k in ('prepare','wait_prepare','worker_wait_issue','stage.acquire_wait','stage.host_copy','launch_publish')})" >> gpurun_out/exp34.log 2>&1
done; done
