mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-restore --nccl-steps 0 --bulk-reps 3 --steps 300"
for defs in "-DKV_UNROLL=8 -DKV_MIN_BLOCKS=3" "-DKV_UNROLL=8 -DKV_MIN_BLOCKS=4" "-DKV_UNROLL=4 -DKV_MIN_BLOCKS=4" "-DKV_UNROLL=16 -DKV_MIN_BLOCKS=2"; do
  KVRING_NVCC_DEFS="$defs" python -c "from paper_2601_22438_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  echo "== $defs" >> gpurun_out/exp4.log
  timeout 300 $B 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['ring_put_kernel_us'], d['step_overhead_us']['median'], d['roofline']['frac'], d['bulk']['roofline']['frac'])" >> gpurun_out/exp4.log 2>&1
done
python -c "from paper_2601_22438_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "not multigpu" > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
