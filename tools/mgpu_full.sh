#!/bin/bash
# Everything multi-GPU on an N-GPU box: parity tests, bench at N, C4 failover at N.
N=${1:-8}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/mgpu_tests_$N.log 2>&1; echo rc=$? >> gpurun_out/mgpu_tests_$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus $N > gpurun_out/bench_n$N.log 2>&1; echo rc=$? >> gpurun_out/bench_n$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29561 tools/c4_failover.py > gpurun_out/c4_n$N.log 2>&1; echo rc=$? >> gpurun_out/c4_n$N.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29563 bench.py --gpus $N --impl reference --steps 20 > gpurun_out/bench_ref_n$N.log 2>&1; echo rc=$? >> gpurun_out/bench_ref_n$N.log
