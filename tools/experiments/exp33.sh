# NVLink counters for the ring-put (single process, stages on GPU 0, successors on GPU 1)
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
python tools/nvlink_profile.py > gpurun_out/nvlink_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes.sum --clock-control none \
    -k regex:kv_ring_put -s 205 -c 30 --csv --log-file gpurun_out/nvlink_ringput.csv python tools/nvlink_profile.py > gpurun_out/nvlink_ncu.log 2>&1
