# ncu of the fused single-launch loop kernel (append k + ring-put k-1), whole-item tasks
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
CMD="python bench.py --loop fused --steps 40 --warmup 3 --e2e-steps 0 --nccl-steps 0 --no-cpu-baseline --no-restore --bulk-reps 0 --interference-steps 0 --block-steps 0 --shared-steps 0"
KVRING_MIN_TASK_SEGS=128 $CMD > gpurun_out/exp26_plain.log 2>&1 || exit 1
KVRING_MIN_TASK_SEGS=128 ncu --set full --clock-control none --import-source on -k regex:kv_step_fused -s 10 -c 2 -o gpurun_out/fused_r01f -f $CMD > gpurun_out/exp26_ncu.log 2>&1
ncu -i gpurun_out/fused_r01f.ncu-rep --page raw --csv > gpurun_out/fused_r01f_raw.csv 2>/dev/null
ncu -i gpurun_out/fused_r01f.ncu-rep --page details > gpurun_out/fused_r01f_details.txt 2>/dev/null
ncu -i gpurun_out/fused_r01f.ncu-rep --page source --csv > gpurun_out/fused_r01f_source.csv 2>/dev/null
