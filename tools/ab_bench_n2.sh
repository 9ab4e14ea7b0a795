#!/bin/bash
# 2-GPU interleaved A/B (gpurun --gpus 2): tools/ab_bench_n2.sh <reps> <name>...
set -u
cd "$(dirname "$0")/.."
LIB=paper_2601_22438_b200/libkvring.so
reps=$1; shift
mkdir -p gpurun_out
cp $LIB _ab/libkvring_default.so
for r in $(seq 1 $reps); do
  for v in "$@"; do
    cp _ab/libkvring_$v.so $LIB
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port $((29700 + r)) bench.py --gpus 2 --steps ${AB_STEPS:-20} --warmup 5 --no-restore \
      --bulk-reps ${AB_BULK:-0} --c4-restores 0 --interference-steps 0 --block-steps 0 \
      --nccl-steps 0 --shared-steps 0 --e2e-steps 0 --no-survey-layout \
      > gpurun_out/abn2_${v}_s${AB_STEPS:-20}_$r.jsonl 2> gpurun_out/abn2_${v}_s${AB_STEPS:-20}_$r.err
    python - "gpurun_out/abn2_${v}_s${AB_STEPS:-20}_$r.jsonl" "$v" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    b = (d.get("bulk") or {}).get("kernel_ms_median")
    print(f"{sys.argv[2]:10s} {d['value']:8.1f} GB/s  {d['ms_per_step']*1e3:6.2f} us/step  "
          f"nvlink frac {d['roofline']['frac']:.4f}" + (f"  bulk {b} ms" if b else ""))
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
  done
done
cp _ab/libkvring_default.so $LIB
