#!/bin/bash
# Multi-GPU checks on an N-GPU box: parity worker + bench at N.
N=${1:-2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/mgpu_tests_$N.log 2>&1; echo rc=$? >> gpurun_out/mgpu_tests_$N.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus $N --steps 300 --warmup 5 > gpurun_out/bench_n$N.log 2>&1; echo rc=$? >> gpurun_out/bench_n$N.log
