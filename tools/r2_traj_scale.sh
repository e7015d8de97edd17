# round 2: B = 1 trajectory parity at scale (many instances per config and mode)
mkdir -p gpurun_out/trs
timeout 3000 python tools/trajectory_scale.py 4 > gpurun_out/trs/result.jsonl 2> gpurun_out/trs/err.log
cat gpurun_out/trs/result.jsonl; tail -3 gpurun_out/trs/err.log
