# N=2: split publication in the graph loop (parity + A/B)
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests/test_multigpu.py -x -q -k "graph" > gpurun_out/exp45_mgpu.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "graph" >> gpurun_out/exp45_mgpu.log 2>&1
B="bench.py --gpus 4 --no-cpu-baseline --e2e-steps 0 --no-restore --nccl-steps 0 --bulk-reps 0 --interference-steps 0 --block-steps 0 --shared-steps 0 --steps 300"
for r in 1 2; do
for v in "X=1" "KVRING_GRAPH_SPLIT_PUB=0"; do
  echo "== $v round $r" >> gpurun_out/exp45.log
  env $v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29585 $B 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['kernel_us']['median'], d['kernel_us']['avg'], d['roofline']['frac'])" >> gpurun_out/exp45.log 2>&1
done; done
