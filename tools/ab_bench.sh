#!/bin/bash
# Interleaved A/B of libkvring builds on ONE box (gpurun, one GPU), from the repo root:
#   tools/ab_bench.sh build <name> "<-D defines>"   (here: build a variant into _ab/)
#   tools/ab_bench.sh run <reps> <name>...          (on the box: bench each variant in turn)
# Each run is the driver's command with the side legs off; the default build is
# restored at the end.
set -u
cd "$(dirname "$0")/.."
LIB=paper_2601_22438_b200/libkvring.so
case "$1" in
build)
  mkdir -p _ab
  KVRING_NVCC_DEFS="$3" python -m paper_2601_22438_b200.build --force > /dev/null
  cp $LIB _ab/libkvring_$2.so
  python -m paper_2601_22438_b200.build --force > /dev/null
  ;;
run)
  reps=$2; shift 2
  mkdir -p gpurun_out
  cp $LIB _ab/libkvring_default.so
  for r in $(seq 1 $reps); do
    for v in "$@"; do
      cp _ab/libkvring_$v.so $LIB
      python bench.py --steps ${AB_STEPS:-20} --warmup 5 --no-cpu-baseline --no-restore \
        --bulk-reps ${AB_BULK:-0} --c4-restores 0 --interference-steps 0 --block-steps 0 \
        --nccl-steps 0 --shared-steps 0 --e2e-steps 0 --no-survey-layout \
        > gpurun_out/ab_${v}_s${AB_STEPS:-20}_$r.jsonl 2> gpurun_out/ab_${v}_s${AB_STEPS:-20}_$r.err
      python - "$v" "s${AB_STEPS:-20}_$r" <<'PY'
import json, sys
v, r = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/ab_{v}_{r}.jsonl").read().strip().splitlines()[-1])
    b = (d.get("bulk") or {}).get("kernel_ms_median")
    print(f"{v:12s} rep {r}: {d['value']:8.1f} GB/s  {d['ms_per_step']*1e3:6.2f} us/step  "
          f"frac {d['roofline']['frac']:.4f}  appends-only {d['step_overhead_us']['step_us_appends_only']:6.2f} us"
          + (f"  bulk {b} ms" if b else ""))
except Exception as e:
    print(v, r, "failed", e)
PY
    done
  done
  cp _ab/libkvring_default.so $LIB
  ;;
esac
