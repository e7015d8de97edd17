# round 2 final set (phase B per eight positions in the large-project kernel):
# GPU tests, smoke, default bench line, reference arm, launch list, ncu of the headline
mkdir -p gpurun_out/fin8
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin8/gpu_tests.log 2>&1
tail -2 gpurun_out/fin8/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin8/smoke.log 2>&1; tail -1 gpurun_out/fin8/smoke.log
( time timeout 1500 python bench.py --steps 20 --warmup 5 ) > gpurun_out/fin8/bench.log 2>&1
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/fin8/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin8/launches.csv python bench.py --steps 1 --warmup 1 --iters 200 --no-cpu-baseline --no-quality --e2e-steps 0 --no-per-config > gpurun_out/fin8/ncu_launch_bench.log 2>&1
python tools/launch_table.py gpurun_out/fin8/launches.csv > gpurun_out/fin8/launches.txt 2>&1
N="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-quality --e2e-steps 0 --no-per-config"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/fin8/k_solve_time $N --instances 148 --iters 150 > gpurun_out/fin8/ncu_time.log 2>&1
python tools/ncu_summary.py gpurun_out/fin8/k_solve_time.ncu-rep > gpurun_out/fin8/k_solve_time.txt 2>&1
python tools/ncu_lines.py gpurun_out/fin8/k_solve_time.ncu-rep 60 > gpurun_out/fin8/k_solve_time_lines.txt 2>&1
