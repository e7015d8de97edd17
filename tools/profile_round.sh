# Round-end measurement set: default bench line, launch list (ncu, cold-cache
# serialised shares), one ncu --set full capture of k_solve, per-config sweep.
set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --iters 200 --no-cpu-baseline --no-quality --e2e-steps 0 > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/k_solve_final python bench.py --instances 148 --steps 1 --warmup 0 --iters 150 --no-cpu-baseline --e2e-steps 0 --no-quality > gpurun_out/ncu_final.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
ls -la gpurun_out
