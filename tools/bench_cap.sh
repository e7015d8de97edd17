# CAPACITY evaluator sweep: warp (group 32, prefix reuse) vs thread per schedule (group 1)
mkdir -p gpurun_out
for cfg in j120 act300; do
 it=1000; [ $cfg = act300 ] && it=100
 for g in 32 1; do
  timeout 300 python bench.py --config $cfg --mode capacity --cap-group $g --iters $it --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bcap_${cfg}_${g}.log 2>&1
  python - <<PY
import json
try:
    d = json.loads(open('gpurun_out/bcap_${cfg}_${g}.log').read().strip().splitlines()[-1])
    print('$cfg cap_group=$g', round(d['value']/1e6, 2), 'M/s  ms/step', round(d['ms_per_step']), 'steps/sched', round(d['roofline']['sgs_steps_per_schedule'], 1))
except Exception as e:
    print('$cfg cap_group=$g FAILED', open('gpurun_out/bcap_${cfg}_${g}.log').read()[-400:])
PY
 done
done
