#!/bin/bash
# ncu evidence for the decode-step kernel (run under gpurun, one GPU):
#   plain runs of tools/step_probe.py, then one `ncu --set full` capture of 4 decode-step
#   launches (the prelude's 399 launches and the first 7 loop launches skipped).
set -x
mkdir -p gpurun_out
tag=${1:-p}
python tools/step_probe.py decode 12 > gpurun_out/${tag}_decode.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:kv_step -s 406 -c 4 \
    -o gpurun_out/${tag}_decode python tools/step_probe.py decode 12 > gpurun_out/${tag}_decode_ncu.log 2>&1
python tools/step_probe.py bulk 4 > gpurun_out/${tag}_bulk.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:kv_step -s 10 -c 1 \
    -o gpurun_out/${tag}_bulk python tools/step_probe.py bulk 4 > gpurun_out/${tag}_bulk_ncu.log 2>&1
