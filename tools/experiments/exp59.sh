# final 1-GPU bench lines with the clock sampler live before the timed region
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for r in 1 2 3; do timeout 600 python bench.py > gpurun_out/exp59_bench_$r.jsonl 2> gpurun_out/exp59_bench_$r.err; done
