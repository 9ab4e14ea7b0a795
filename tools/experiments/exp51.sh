# graph structure A/B without timing events: default vs lean (no timing nodes)
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
KVRING_GRAPH_LEAN=1 timeout 600 python -m pytest tests -m gpu -x -q -k "graph_bit_exact" > gpurun_out/exp51_tests.log 2>&1
for r in 1 2 3; do
for v in "X=1" "KVRING_GRAPH_LEAN=1"; do
  echo "== $v round $r" >> gpurun_out/exp51.log
  env $v timeout 300 python tools/graph_ab.py >> gpurun_out/exp51.log 2>&1
done; done
