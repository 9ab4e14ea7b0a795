# N=2 e2e leg reproducibility
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
B="bench.py --gpus 2 --no-cpu-baseline --no-restore --nccl-steps 0 --bulk-reps 0 --interference-steps 0 --block-steps 0 --shared-steps 0 --steps 100"
for r in 1 2; do
  echo "== round $r" >> gpurun_out/exp31.log
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29577 $B 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e'])" >> gpurun_out/exp31.log 2>&1
done
echo "== N=1" >> gpurun_out/exp31.log
timeout 300 python bench.py --no-cpu-baseline --no-restore --nccl-steps 0 --bulk-reps 0 --interference-steps 0 --block-steps 0 --shared-steps 0 --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e'])" >> gpurun_out/exp31.log 2>&1
