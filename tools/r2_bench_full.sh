mkdir -p gpurun_out/bf
( time timeout 1500 python bench.py --steps 20 --warmup 5 ) > gpurun_out/bf/bench.log 2>&1
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/bf/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bf/launches.csv python bench.py --steps 1 --warmup 1 --iters 200 --no-cpu-baseline --no-quality --e2e-steps 0 --no-per-config > gpurun_out/bf/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/bf/k_solve_j120p python bench.py --instances 148 --steps 1 --warmup 0 --iters 150 --no-cpu-baseline --e2e-steps 0 --no-quality --no-per-config > gpurun_out/bf/ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/bf/k_solve_j120p.ncu-rep > gpurun_out/bf/k_solve_j120p.txt 2>&1
python tools/ncu_lines.py gpurun_out/bf/k_solve_j120p.ncu-rep 60 > gpurun_out/bf/k_solve_j120p_lines.txt 2>&1
