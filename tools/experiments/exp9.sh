mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
B="bench.py --gpus 2 --no-cpu-baseline --e2e-steps 0 --no-restore --nccl-steps 0 --bulk-reps 2 --interference-steps 0 --block-steps 0 --steps 300"
for v in "X=1" "KVRING_DEBUG_RINGPUT_NOPUB=1"; do
  echo "== $v" >> gpurun_out/exp9.log
  env $v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29557 $B 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['ring_put_kernel_us'], d['roofline']['frac'], d['bulk']['roofline']['frac']); print(d['host_us_per_step'])" >> gpurun_out/exp9.log 2>&1
done
