# round 2: ncu --set full of the CAPACITY kernel on 300 activities (current)
mkdir -p gpurun_out/p6
N="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-quality --e2e-steps 0 --no-per-config"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/p6/cap_act300 $N --config act300 --mode capacity --instances 148 --workers 2 --iters 30 > gpurun_out/p6/ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/p6/cap_act300.ncu-rep > gpurun_out/p6/cap_act300.txt 2>&1
python tools/ncu_lines.py gpurun_out/p6/cap_act300.ncu-rep 3000 > gpurun_out/p6/cap_act300_lines.txt 2>&1
