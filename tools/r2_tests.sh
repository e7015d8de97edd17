mkdir -p gpurun_out/t
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t/gpu_tests.log 2>&1
tail -3 gpurun_out/t/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t/smoke.log 2>&1; tail -1 gpurun_out/t/smoke.log
