mkdir -p gpurun_out/rr
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/rr/gpu_tests.log 2>&1
tail -3 gpurun_out/rr/gpu_tests.log
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-quality --e2e-steps 0 --no-per-config"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/rr/time_j30p $B --config j30p --mode time --instances 148 --workers 8 --iters 1000 > gpurun_out/rr/ncu_time_j30p.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/rr/time_j60p $B --config j60p --mode time --instances 148 --workers 8 --iters 1000 > gpurun_out/rr/ncu_time_j60p.log 2>&1
for r in time_j30p time_j60p; do
  python tools/ncu_summary.py gpurun_out/rr/$r.ncu-rep > gpurun_out/rr/$r.txt 2>&1
  python tools/ncu_lines.py gpurun_out/rr/$r.ncu-rep 60 > gpurun_out/rr/${r}_lines.txt 2>&1
done
bash tools/r2_populations.sh
