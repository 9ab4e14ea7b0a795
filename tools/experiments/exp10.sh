mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "run_steps or c1_bit" > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --no-restore --nccl-steps 0 --bulk-reps 0 --interference-steps 0 --block-steps 0 --steps 200 --timeline > gpurun_out/tl_2s.log 2>&1
