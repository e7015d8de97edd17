# round 2: GPU tests + CAPACITY sweep after the closed-form Alg. 4 evaluator
set -x
mkdir -p gpurun_out/r2
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2/gpu_tests.log 2>&1
tail -5 gpurun_out/r2/gpu_tests.log
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-quality --e2e-steps 0 --no-per-config"
for c in "j120p 600 2 1000" "act300 148 2 100" "j60p 148 8 1000" "j120 600 2 1000" "j60 148 8 1000" "j30 148 8 1000"; do
  set -- $c
  for g in 32 1; do
    timeout 600 $B --config $1 --instances $2 --workers $3 --iters $4 --mode capacity --cap-group $g > gpurun_out/r2/cap_$1_g$g.log 2>&1
    python -c "
import json,sys
try:
  d=json.loads(open('gpurun_out/r2/cap_$1_g$g.log').read().strip().splitlines()[-1]); print('$1 cap g$g', round(d['value']/1e6,2), 'M/s frac', round(d['roofline']['frac'],4), 'steps/sched', round(d['roofline']['sgs_steps_per_schedule'],1), 'cpm', round(d['run']['cpm_dev'],2))
except Exception as e: print('$1 g$g FAILED', open('gpurun_out/r2/cap_$1_g$g.log').read()[-600:])
" | tee -a gpurun_out/r2/cap_summary.txt
  done
done
