# round 2: per-step search times of j30p / j60p / j120p batch solves (bimodality check)
mkdir -p gpurun_out/jit
timeout 600 python tools/step_jitter.py j30p 148 8 1000 40 > gpurun_out/jit/j30p.txt 2>&1
timeout 600 python tools/step_jitter.py j60p 148 8 1000 30 > gpurun_out/jit/j60p.txt 2>&1
timeout 600 python tools/step_jitter.py j120p 600 2 300 10 > gpurun_out/jit/j120p.txt 2>&1
nvidia-smi -q -d CLOCK,PERFORMANCE | head -60 > gpurun_out/jit/smi.txt
cat gpurun_out/jit/*.txt | head -80
