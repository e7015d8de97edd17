# Per-config sweep of the B200 arm (both evaluation modes), one line per run.
mkdir -p gpurun_out/configs
for cfg in j30p j60p j120p j30 j60 j120 act300; do
 for mode in time capacity; do
  it=1000; n=148; [ $cfg = act300 ] && it=300
  [ $cfg = j120p ] && n=600; [ $cfg = j120 ] && n=600
  w=2; case $cfg in j30*|j60*) w=8;; esac
  timeout 400 python bench.py --config $cfg --mode $mode --instances $n --workers $w --iters $it --steps 2 --warmup 2 --no-cpu-baseline --no-quality --e2e-steps 0 > gpurun_out/configs/b_${cfg}_${mode}.log 2>&1
  python - <<PY
import json
try:
    d = json.loads(open('gpurun_out/configs/b_${cfg}_${mode}.log').read().strip().splitlines()[-1])
    print('$cfg $mode', '$n x $w', round(d['value']/1e6, 2), 'M sched/s  ms/step', round(d['ms_per_step']), 'cpm_dev', round(d['config']['cpm_dev'], 2), 'steps/sched', round(d['roofline']['sgs_steps_per_schedule'], 1))
except Exception as e:
    print('$cfg $mode FAILED', open('gpurun_out/configs/b_${cfg}_${mode}.log').read()[-300:])
PY
 done
done
