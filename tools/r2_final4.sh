# round 2: new CAPACITY-beyond-packing test, headline-only launch list
mkdir -p gpurun_out/fin4
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py -k "beyond_time_packing or small_shapes or batch_solve_shapes" > gpurun_out/fin4/tests.log 2>&1
tail -3 gpurun_out/fin4/tests.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin4/launches.csv python bench.py --steps 1 --warmup 1 --iters 200 --no-cpu-baseline --no-quality --e2e-steps 0 --no-per-config > gpurun_out/fin4/ncu_launch_bench.log 2>&1
python tools/launch_table.py gpurun_out/fin4/launches.csv > gpurun_out/fin4/launches.txt 2>&1
cat gpurun_out/fin4/launches.txt
