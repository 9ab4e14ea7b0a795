# N=2: system-scope RMW per CTA vs GPU-scope RMW + one system fence in the completing CTA
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 400 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/mgpu_tests_2.log 2>&1; echo rc=$? >> gpurun_out/mgpu_tests_2.log
B="bench.py --gpus 2 --no-cpu-baseline --e2e-steps 0 --no-restore --nccl-steps 0 --bulk-reps 2 --interference-steps 0 --block-steps 0 --steps 300"
for v in "X=1" "KVRING_SYS_PER_CTA=1" "X=1" "KVRING_SYS_PER_CTA=1"; do
  echo "== $v" >> gpurun_out/exp12.log
  env $v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29557 $B 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['kernel_us'], d['roofline']['frac'], d['bulk']['roofline']['frac'])" >> gpurun_out/exp12.log 2>&1
done
