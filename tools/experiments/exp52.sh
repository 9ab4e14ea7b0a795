# final verification with the step roofline key: build, smoke, GPU suite, two 1-GPU bench lines
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" > gpurun_out/exp52_build.log 2>&1 || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/exp52_smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/exp52_suite.log 2>&1; echo "rc=$?" >> gpurun_out/exp52_suite.log
for r in 1 2; do
  timeout 600 python bench.py > gpurun_out/exp52_bench_$r.jsonl 2> gpurun_out/exp52_bench_$r.err
done
