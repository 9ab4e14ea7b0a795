# fused single-stream loop vs two-stream loop (1 GPU), plus parity of the fused loop
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "not multigpu and not whole" > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-restore --nccl-steps 0 --bulk-reps 0 --interference-steps 0 --block-steps 0 --steps 400"
for v in "--loop streams" "--loop streams"; do
  echo "== $v" >> gpurun_out/exp11.log
  timeout 300 $B $v 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['kernel_us'], d['roofline']['frac']); print(d['host_us_per_step'])" >> gpurun_out/exp11.log 2>&1
done
