# round 2: ncu --set full of the current CAPACITY search kernel (j120p, 148
# instances) with source lines and SASS, to attribute instructions per step
mkdir -p gpurun_out/p4
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-quality --e2e-steps 0 --no-per-config"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/p4/cap_j120p $B --config j120p --mode capacity --instances 148 --iters 100 > gpurun_out/p4/ncu_cap_j120p.log 2>&1
python tools/ncu_summary.py gpurun_out/p4/cap_j120p.ncu-rep > gpurun_out/p4/cap_j120p.txt 2>&1
python tools/ncu_lines.py gpurun_out/p4/cap_j120p.ncu-rep 90 > gpurun_out/p4/cap_j120p_lines.txt 2>&1
ncu -i gpurun_out/p4/cap_j120p.ncu-rep --page source --csv --print-source sass > gpurun_out/p4/cap_j120p_sass.csv 2>/dev/null
ls -la gpurun_out/p4
