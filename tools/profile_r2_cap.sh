# Round 2: ncu --set full captures of the CAPACITY search kernel (j120p, act300)
# and of the TIME kernel on small projects (j30p), plus a config sweep.
set -x
mkdir -p gpurun_out/r2
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-quality --e2e-steps 0"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/r2/cap_j120p $B --config j120p --mode capacity --instances 148 --iters 100 > gpurun_out/r2/ncu_cap_j120p.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/r2/cap_act300 $B --config act300 --mode capacity --instances 148 --iters 30 > gpurun_out/r2/ncu_cap_act300.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/r2/time_j30p $B --config j30p --mode time --instances 296 --workers 8 --iters 300 > gpurun_out/r2/ncu_time_j30p.log 2>&1
for r in cap_j120p cap_act300 time_j30p; do
  python tools/ncu_summary.py gpurun_out/r2/$r.ncu-rep > gpurun_out/r2/$r.txt 2>&1
  python tools/ncu_lines.py gpurun_out/r2/$r.ncu-rep 60 > gpurun_out/r2/${r}_lines.txt 2>&1
done
ls -la gpurun_out/r2
