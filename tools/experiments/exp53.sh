# 2- and 4-GPU bench lines with the step_roofline key (same code as exp52)
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" > gpurun_out/exp53_build.log 2>&1 || exit 1
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 29511 bench.py --gpus $n > gpurun_out/exp53_bench_n$n.jsonl 2> gpurun_out/exp53_bench_n$n.err
done
