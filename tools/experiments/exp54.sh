# CTA size / count vs the ramp of a single-wave copy kernel (tools/ctasize_bench.cu)
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/ctasize_bench tools/ctasize_bench.cu || exit 1
for mb in 8 19 38; do for w in 1 0; do timeout 120 /tmp/ctasize_bench $mb $w; done; done > gpurun_out/exp54.log 2>&1
