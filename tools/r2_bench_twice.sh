mkdir -p gpurun_out/fin9
for r in 1 2; do
( time timeout 1500 python bench.py --steps 20 --warmup 5 ) > gpurun_out/fin9/bench_$r.log 2>&1
done
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/fin9/bench_ref.log 2>&1
