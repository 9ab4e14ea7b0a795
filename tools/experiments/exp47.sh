# graph loop: timing event nodes beside the chain vs in it
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "graph or c2_full or abort" > gpurun_out/exp47_tests.log 2>&1
B="bench.py --no-cpu-baseline --e2e-steps 0 --no-restore --nccl-steps 0 --bulk-reps 0 --interference-steps 0 --block-steps 0 --shared-steps 0 --steps 400"
for r in 1 2 3; do
for v in "X=1" "KVRING_GRAPH_EVENTS_IN_CHAIN=1"; do
  echo "== $v round $r" >> gpurun_out/exp47.log
  env $v timeout 300 python $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['kernel_us']['median'], d['kernel_us']['avg'])" >> gpurun_out/exp47.log 2>&1
done; done
