# graph loop with half-size grids (KVRING_CTAS_PER_SM=2): append k+1 and copy k can co-reside
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
KVRING_CTAS_PER_SM=2 timeout 600 python -m pytest tests -m gpu -x -q -k "graph" > gpurun_out/exp55_tests.log 2>&1
for r in 1 2 3; do
for v in "X=1" "KVRING_CTAS_PER_SM=2" "KVRING_CTAS_PER_SM=3"; do
  echo "== $v round $r" >> gpurun_out/exp55.log
  env $v timeout 300 python tools/graph_ab.py >> gpurun_out/exp55.log 2>&1
done; done
