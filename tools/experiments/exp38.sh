# priority of the ring-put over the concurrent append (graph node attribute / stream priority)
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
B="bench.py --no-cpu-baseline --e2e-steps 0 --no-restore --nccl-steps 0 --bulk-reps 0 --interference-steps 0 --block-steps 0 --shared-steps 0 --steps 400"
for r in 1 2; do
for v in "X=1 graph" "KVRING_GRAPH_PRIO=1 graph" "X=1 streams" "KVRING_REPL_PRIO=1 streams"; do
  set -- $v
  echo "== $v round $r" >> gpurun_out/exp38.log
  env $1 timeout 300 python $B --loop $2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['kernel_us']['median'], d['kernel_us']['avg'])" >> gpurun_out/exp38.log 2>&1
done; done
