# final 1-GPU bench lines (population traffic in roofline) + reference arm
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for r in 1 2; do timeout 600 python bench.py > gpurun_out/exp58_bench_$r.jsonl 2> gpurun_out/exp58_bench_$r.err; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/exp58_ref.jsonl 2> gpurun_out/exp58_ref.err
