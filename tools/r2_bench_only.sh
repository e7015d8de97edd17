mkdir -p gpurun_out/fin7
( time timeout 1500 python bench.py --steps 20 --warmup 5 ) > gpurun_out/fin7/bench.log 2>&1
tail -4 gpurun_out/fin7/bench.log | head -1 | cut -c1-300
