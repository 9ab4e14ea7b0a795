# graph loop: steps per graph
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
KVRING_GRAPH_STEPS=16 timeout 600 python -m pytest tests -m gpu -x -q -k "graph" > gpurun_out/exp42_tests.log 2>&1
KVRING_GRAPH_STEPS=3 timeout 600 python -m pytest tests -m gpu -x -q -k "graph" >> gpurun_out/exp42_tests.log 2>&1
B="bench.py --no-cpu-baseline --e2e-steps 0 --no-restore --nccl-steps 0 --bulk-reps 0 --interference-steps 0 --block-steps 0 --shared-steps 0 --steps 400"
for r in 1 2; do
for v in 8 4 16 32; do
  echo "== G=$v round $r" >> gpurun_out/exp42.log
  KVRING_GRAPH_STEPS=$v timeout 300 python $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['kernel_us']['median'], d['kernel_us']['avg'])" >> gpurun_out/exp42.log 2>&1
done; done
