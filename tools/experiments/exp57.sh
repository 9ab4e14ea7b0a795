# ncu --set full over a POPULATION of graph copy-node launches (C2 decode steps, warm-up + timed
# steps of the default loop): per-launch DRAM traffic next to the L2 bytes the kernel requested
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
CMD="python bench.py --steps 40 --warmup 3 --e2e-steps 0 --nccl-steps 0 --no-cpu-baseline --no-restore --bulk-reps 0 --interference-steps 0 --block-steps 0 --shared-steps 0"
$CMD > gpurun_out/exp57_plain.log 2>&1 || exit 1
M="dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,gpu__time_duration.sum"
timeout 1500 ncu --set full --metrics $M --clock-control none -k regex:kv_ring_put_copy -c 32 -o gpurun_out/copynode_pop_r01 -f $CMD > gpurun_out/exp57_ncu.log 2>&1
ncu -i gpurun_out/copynode_pop_r01.ncu-rep --page raw --csv --metrics $M > gpurun_out/copynode_pop_r01_raw.csv 2>/dev/null
