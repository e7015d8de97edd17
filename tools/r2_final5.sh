# round 2 final bench set after the CAPACITY launch-bound change
mkdir -p gpurun_out/fin5
( time timeout 1500 python bench.py --steps 20 --warmup 5 ) > gpurun_out/fin5/bench.log 2>&1
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/fin5/bench_ref.log 2>&1
B2="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-quality --e2e-steps 0 --no-per-config"
for c in "act300 148 2 100 time" "act300 148 2 100 capacity" "j120p 600 2 1000 capacity" "j60p 148 8 1000 capacity" "j30p 148 8 1000 capacity" "j120 600 2 1000 capacity" "j60 148 8 1000 capacity" "j30 148 8 1000 capacity" "j30p 148 8 1000 time" "j60p 148 8 1000 time" "j30 148 8 1000 time" "j60 148 8 1000 time" "j120 600 2 1000 time"; do
  set -- $c
  timeout 600 $B2 --config $1 --instances $2 --workers $3 --iters $4 --mode $5 > gpurun_out/fin5/b_$1_$5.log 2>&1
  python -c "
import json
try:
  d=json.loads(open('gpurun_out/fin5/b_$1_$5.log').read().strip().splitlines()[-1]); print('$1 $5', round(d['value']/1e6,2), 'M/s frac', round(d['roofline']['frac'],4), 'steps/sched', round(d['roofline']['sgs_steps_per_schedule'],1), 'cpm', round(d['run']['cpm_dev'],2))
except Exception as e: print('$1 $5 FAILED', open('gpurun_out/fin5/b_$1_$5.log').read()[-600:])
" | tee -a gpurun_out/fin5/summary.txt
done
