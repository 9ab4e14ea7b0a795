# e2e leg with zero-copy pinned host sources (N=1 default window and N=2)
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "host_source or run_steps or c1" > gpurun_out/exp32_tests.log 2>&1
B="--no-cpu-baseline --no-restore --nccl-steps 0 --bulk-reps 0 --interference-steps 0 --block-steps 0 --shared-steps 0"
timeout 300 python bench.py $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('N=1', d['value'], d['e2e'])" >> gpurun_out/exp32.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29579 bench.py --gpus 2 $B 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('N=2', d['value'], d['e2e'])" >> gpurun_out/exp32.log 2>&1
