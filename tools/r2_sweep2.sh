# round 2 final: GPU tests, per-config sweep (TIME and CAPACITY), mode-rule re-derivation
mkdir -p gpurun_out/sw2
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/sw2/gpu_tests.log 2>&1
tail -2 gpurun_out/sw2/gpu_tests.log
B2="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-quality --e2e-steps 0 --no-per-config"
for c in "act300 148 2 100 time" "act300 148 2 100 capacity" "j120p 600 2 1000 time" "j120p 600 2 1000 capacity" "j60p 148 8 1000 time" "j60p 148 8 1000 capacity" "j30p 148 8 1000 time" "j30p 148 8 1000 capacity" "j120 600 2 1000 time" "j60 148 8 1000 time" "j30 148 8 1000 time"; do
  set -- $c
  timeout 600 $B2 --config $1 --instances $2 --workers $3 --iters $4 --mode $5 > gpurun_out/sw2/b_$1_$5.log 2>&1
  python -c "
import json
try:
  d=json.loads(open('gpurun_out/sw2/b_$1_$5.log').read().strip().splitlines()[-1]); print('$1 $5', round(d['value']/1e6,2), 'M/s frac', round(d['roofline']['frac'],4), 'steps/sched', round(d['roofline']['sgs_steps_per_schedule'],1), 'cpm', round(d['run']['cpm_dev'],2))
except Exception as e: print('$1 $5 FAILED', open('gpurun_out/sw2/b_$1_$5.log').read()[-600:])
" | tee -a gpurun_out/sw2/summary.txt
done
for c in "j120 600 2 1000" "j60 148 8 1000" "j30 148 8 1000"; do
  set -- $c
  timeout 600 $B2 --config $1 --instances $2 --workers $3 --iters $4 --mode capacity > gpurun_out/sw2/c_$1.log 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/sw2/c_$1.log').read().strip().splitlines()[-1]); print('$1 capacity', round(d['value']/1e6,2), 'M/s frac', round(d['roofline']['frac'],4), 'steps/sched', round(d['roofline']['sgs_steps_per_schedule'],1))
" | tee -a gpurun_out/sw2/summary.txt
done
timeout 1200 python tools/derive_rules.py --out gpurun_out/sw2/mode_rules_b200.json > gpurun_out/sw2/derive_rules.log 2>&1
cat gpurun_out/sw2/derive_rules.log
