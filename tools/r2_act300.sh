mkdir -p gpurun_out/a3
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-quality --e2e-steps 0 --no-per-config"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/a3/time_act300 $B --config act300 --mode time --instances 148 --iters 60 > gpurun_out/a3/ncu_time_act300.log 2>&1
python tools/ncu_summary.py gpurun_out/a3/time_act300.ncu-rep > gpurun_out/a3/time_act300.txt 2>&1
python tools/ncu_lines.py gpurun_out/a3/time_act300.ncu-rep 50 > gpurun_out/a3/time_act300_lines.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/a3/cap_act300 $B --config act300 --mode capacity --instances 148 --iters 30 > gpurun_out/a3/ncu_cap_act300.log 2>&1
python tools/ncu_summary.py gpurun_out/a3/cap_act300.ncu-rep > gpurun_out/a3/cap_act300.txt 2>&1
python tools/ncu_lines.py gpurun_out/a3/cap_act300.ncu-rep 50 > gpurun_out/a3/cap_act300_lines.txt 2>&1
