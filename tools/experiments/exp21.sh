# interleaved A/B (3 rounds): inline size classes vs staged, task size 64 vs 128 segs
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "run_steps or pdl or c2 or ragged" > gpurun_out/exp21_tests.log 2>&1
B="bench.py --no-cpu-baseline --e2e-steps 0 --no-restore --nccl-steps 0 --bulk-reps 0 --interference-steps 0 --block-steps 0 --shared-steps 0 --steps 400"
for r in 1 2 3; do
for v in "X=1" "KVRING_INLINE=0" "KVRING_MIN_TASK_SEGS=128" "KVRING_INLINE=0,KVRING_MIN_TASK_SEGS=128"; do
  echo "== $v round $r" >> gpurun_out/exp21.log
  env $(echo $v | tr ',' ' ') timeout 300 python $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['kernel_us']['median'], d['roofline']['frac'], d['clocks']['sm_mhz'], {k: d['host_us_per_step'][k] for k in ('prepare','wait_prepare','stage_h2d','launch_append','launch_publish')})" >> gpurun_out/exp21.log 2>&1
done; done
