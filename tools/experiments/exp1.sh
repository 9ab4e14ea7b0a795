mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-restore --steps 300"
for v in "X=1" "KVRING_DEBUG_RINGPUT_NOPUB=1" "KVRING_CTAS_PER_SM=4" "KVRING_CTAS_PER_SM=2" "KVRING_CTAS_PER_SM=16"; do
  echo "== $v" >> gpurun_out/exp1.log
  env $v $B 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['ring_put_kernel_us'], d['step_overhead_us']['median'], d['roofline']['frac'])" >> gpurun_out/exp1.log 2>&1
done
