#!/bin/bash
# 2-GPU checks (gpurun --gpus 2): the multi-GPU parity tests, the R9 concurrent-reader
# worker with its summary line, and a short 2-GPU bench line.
tag=${1:-m}
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q -x > gpurun_out/${tag}_tests.log 2>&1; echo tests rc=$?
KV_TRANSPORT=r9 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 tests/mgpu_worker.py > gpurun_out/${tag}_r9.log 2>&1; echo r9 rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/${tag}_bench20.jsonl 2> gpurun_out/${tag}_bench20.err; echo bench rc=$?
