#!/bin/bash
# 4-GPU checks (gpurun --gpus 4): multi-GPU parity tests, the C4 failover tool at N=4,
# and the bench at N=4 (weak layout + the SURVEY §8(e) one-stage-per-GPU layout).
tag=${1:-m4}
timeout 1200 python -m pytest tests/test_multigpu.py -m gpu -q > gpurun_out/${tag}_tests.log 2>&1; echo tests rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/${tag}_bench20.jsonl 2> gpurun_out/${tag}_bench20.err; echo bench rc=$?
