mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-restore --nccl-steps 0 --bulk-reps 0 --steps 200 --timeline"
timeout 300 $B > gpurun_out/tl_2s.log 2>&1
timeout 300 $B --single-stream > gpurun_out/tl_1s.log 2>&1
