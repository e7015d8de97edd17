mkdir -p gpurun_out/dyn
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py -k "decide_dynamic or beyond_time_packing" > gpurun_out/dyn/tests.log 2>&1
tail -15 gpurun_out/dyn/tests.log
