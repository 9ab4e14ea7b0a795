# fixed-node (self-describing) graph steps: parity + A/B
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
KVRING_GRAPH_FIXED=1 timeout 900 python -m pytest tests -m gpu -x -q -k "graph or c2_full or abort" > gpurun_out/exp49_tests.log 2>&1
B="bench.py --no-cpu-baseline --e2e-steps 0 --no-restore --nccl-steps 0 --bulk-reps 0 --interference-steps 0 --block-steps 0 --shared-steps 0 --steps 400"
for r in 1 2 3; do
for v in "X=1" "KVRING_GRAPH_FIXED=1"; do
  echo "== $v round $r" >> gpurun_out/exp49.log
  env $v timeout 300 python $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); h=d['host_us_per_step']; print(d['value'], d['ms_per_step'], d['kernel_us']['median'], d['kernel_us']['avg'], {k: h[k] for k in ('prepare','wait_prepare','launch_publish','stage.host_copy','stage.acquire_wait','worker_wait_issue')})" >> gpurun_out/exp49.log 2>&1
done; done
