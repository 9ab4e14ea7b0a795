mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "not multigpu" > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-restore --nccl-steps 0 --bulk-reps 3 --steps 300"
for v in "X=1" "KVRING_DEBUG_RINGPUT_NOPUB=1"; do
  for ss in "" "--single-stream"; do
  echo "== $v $ss" >> gpurun_out/exp3.log
  env $v timeout 300 $B $ss 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['wall_s_timed'], d['ring_put_kernel_us'], d['step_overhead_us']['median'], d['roofline']['frac'], d['bulk']['roofline']['frac'])" >> gpurun_out/exp3.log 2>&1
  done
done
CMD="python bench.py --steps 40 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-restore --nccl-steps 0 --bulk-reps 2 --single-stream"
timeout 300 $CMD > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:kv_ --csv --log-file gpurun_out/launches_r01d.csv $CMD > /dev/null 2>&1
echo done
