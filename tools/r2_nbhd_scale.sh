# round 2: neighbourhood parity at scale (>= 1e7 moves per config and mode)
mkdir -p gpurun_out/nbs
timeout 3000 python tools/neighbourhood_scale.py 1e7 > gpurun_out/nbs/result.jsonl 2> gpurun_out/nbs/err.log
cat gpurun_out/nbs/result.jsonl; tail -3 gpurun_out/nbs/err.log
