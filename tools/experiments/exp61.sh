# final GPU suite on 4 GPUs (the multi-GPU tests run) with the session's final code
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" > gpurun_out/exp61_build.log 2>&1 || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/exp61_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/exp61_suite.log 2>&1; echo "rc=$?" >> gpurun_out/exp61_suite.log
