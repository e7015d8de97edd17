# round 2: ncu of the closed-form CAPACITY evaluator + TIME j30p at the bench shape; sanitizer
set -x
mkdir -p gpurun_out/r2b
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-quality --e2e-steps 0 --no-per-config"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/r2b/cap_j120p $B --config j120p --mode capacity --instances 148 --iters 100 > gpurun_out/r2b/ncu_cap_j120p.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/r2b/time_j30p $B --config j30p --mode time --instances 148 --workers 8 --iters 1000 > gpurun_out/r2b/ncu_time_j30p.log 2>&1
for r in cap_j120p time_j30p; do
  python tools/ncu_summary.py gpurun_out/r2b/$r.ncu-rep > gpurun_out/r2b/$r.txt 2>&1
  python tools/ncu_lines.py gpurun_out/r2b/$r.ncu-rep 60 > gpurun_out/r2b/${r}_lines.txt 2>&1
done
bash tools/r2_sanitize.sh
