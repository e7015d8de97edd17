# round 2: ncu --set full of the TIME search kernel on j30p at the bench shape
# (148 x 8 CTAs, 1000 iterations) after the out-of-line evaluator dispatch
mkdir -p gpurun_out/p5
N="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-quality --e2e-steps 0 --no-per-config"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/p5/time_j30p $N --config j30p --mode time --instances 148 --workers 8 --iters 1000 > gpurun_out/p5/ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/p5/time_j30p.ncu-rep > gpurun_out/p5/time_j30p.txt 2>&1
python tools/ncu_lines.py gpurun_out/p5/time_j30p.ncu-rep 3000 > gpurun_out/p5/time_j30p_lines.txt 2>&1
