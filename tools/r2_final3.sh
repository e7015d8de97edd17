# round 2 final set (after the CAPACITY register rows and the out-of-line
# evaluator dispatch): GPU tests, default bench line, reference arm, smoke,
# launch list, ncu --set full of k_solve (TIME, headline shape) and of the
# CAPACITY kernel
mkdir -p gpurun_out/fin3
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin3/gpu_tests.log 2>&1
tail -2 gpurun_out/fin3/gpu_tests.log
( time timeout 1500 python bench.py --steps 20 --warmup 5 ) > gpurun_out/fin3/bench.log 2>&1
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/fin3/bench_ref.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin3/smoke.log 2>&1
tail -1 gpurun_out/fin3/smoke.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin3/launches.csv python bench.py --steps 1 --warmup 1 --iters 200 --no-cpu-baseline --no-quality --e2e-steps 0 > gpurun_out/fin3/ncu_launch_bench.log 2>&1
N="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-quality --e2e-steps 0 --no-per-config"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/fin3/k_solve_time $N --instances 148 --iters 150 > gpurun_out/fin3/ncu_time.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/fin3/k_solve_cap $N --config j120p --mode capacity --instances 148 --iters 100 > gpurun_out/fin3/ncu_cap.log 2>&1
for r in k_solve_time k_solve_cap; do
  python tools/ncu_summary.py gpurun_out/fin3/$r.ncu-rep > gpurun_out/fin3/$r.txt 2>&1
  python tools/ncu_lines.py gpurun_out/fin3/$r.ncu-rep 60 > gpurun_out/fin3/${r}_lines.txt 2>&1
done
ls -la gpurun_out/fin3
