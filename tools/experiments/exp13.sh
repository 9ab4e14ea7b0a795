# timeline of both streams (append / ring-put) at N=1 with grid knobs
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
B="bench.py --no-cpu-baseline --e2e-steps 0 --no-restore --nccl-steps 0 --bulk-reps 0 --interference-steps 0 --block-steps 0 --steps 400"
for v in "X=1" "KVRING_CTAS_PER_SM=2" "KVRING_CTAS_PER_SM=3"; do
  echo "== $v" >> gpurun_out/exp13.log
  env $v timeout 300 python $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['ring_put_kernel_us'], d['roofline']['frac']); print(d['host_us_per_step'])" >> gpurun_out/exp13.log 2>&1
  env $v timeout 300 python $B --timeline 2>> gpurun_out/exp13_timeline_$v.log >/dev/null
done
