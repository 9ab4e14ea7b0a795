# PDL single-stream loop with inline (parameter-space) descriptors vs zero-copy vs streams
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "pdl or fused or two_streams" > gpurun_out/exp14_tests.log 2>&1
B="bench.py --no-cpu-baseline --e2e-steps 0 --no-restore --nccl-steps 0 --bulk-reps 0 --interference-steps 0 --block-steps 0 --steps 400"
for v in "X=1 --loop streams" "X=1 --loop pdl" "KVRING_INLINE=0 --loop pdl"; do
  set -- $v
  echo "== $v" >> gpurun_out/exp14.log
  env $1 timeout 300 python $B $2 $3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['kernel_us'], d['roofline']['frac']); print(d['host_us_per_step'])" >> gpurun_out/exp14.log 2>&1
done
timeout 300 python $B --loop pdl --timeline 2> gpurun_out/exp14_timeline_pdl.log >/dev/null
