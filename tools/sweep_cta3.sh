for cfg in j30 j60; do
for w in 2 4 8; do
  timeout 300 python bench.py --config $cfg --instances 148 --workers $w --steps 2 --warmup 3 --no-cpu-baseline --no-quality --e2e-steps 0 > gpurun_out/sc.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/sc.log').read().strip().splitlines()[-1]); print('$cfg auto threads, workers $w', round(d['value']/1e6,2), 'ms/step', round(d['ms_per_step']))" || tail -2 gpurun_out/sc.log
done; done
