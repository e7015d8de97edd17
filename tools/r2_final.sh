mkdir -p gpurun_out/fin
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin/gpu_tests.log 2>&1
tail -2 gpurun_out/fin/gpu_tests.log
( time timeout 1500 python bench.py --steps 20 --warmup 5 ) > gpurun_out/fin/bench.log 2>&1
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/fin/bench_ref.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1
tail -1 gpurun_out/fin/smoke.log
