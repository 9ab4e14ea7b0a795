# ncu capture of the restore kernel (local restore of a batch-64 stage, C2) and a C5 bulk copy node
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
CMD="python bench.py --steps 20 --warmup 3 --e2e-steps 0 --nccl-steps 0 --no-cpu-baseline --bulk-reps 1 --interference-steps 0 --block-steps 0 --shared-steps 0"
$CMD > gpurun_out/exp50_plain.log 2>&1 || exit 1
ncu --set full --clock-control none -k regex:kv_restore_remap -c 1 -o gpurun_out/restore_r01 -f $CMD > gpurun_out/exp50_ncu.log 2>&1
ncu -i gpurun_out/restore_r01.ncu-rep --page raw --csv > gpurun_out/restore_r01_raw.csv 2>/dev/null
