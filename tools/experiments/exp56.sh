# parallel per-pool host prepare in the graph loop (KVRING_GRAPH_PAR_PREP=1): parity + A/B
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" > gpurun_out/exp56_build.log 2>&1 || exit 1
KVRING_GRAPH_PAR_PREP=1 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/exp56_tests.log 2>&1; echo "rc=$?" >> gpurun_out/exp56_tests.log
for r in 1 2 3; do
for v in "X=1" "KVRING_GRAPH_PAR_PREP=1" "KVRING_GRAPH_PAR_PREP=1 KVRING_CTAS_PER_SM=2"; do
  echo "== $v round $r" >> gpurun_out/exp56.log
  env $v timeout 300 python tools/graph_ab.py >> gpurun_out/exp56.log 2>&1
done; done
KVRING_GRAPH_PAR_PREP=1 timeout 600 python bench.py > gpurun_out/exp56_bench.jsonl 2> gpurun_out/exp56_bench.err
