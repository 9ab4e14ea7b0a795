python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
python -m cProfile -s cumtime bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-restore --nccl-steps 0 --bulk-reps 0 --interference-steps 0 --block-steps 0 --shared-steps 0 --e2e-steps 200 > gpurun_out/e2e_prof.log 2>&1
