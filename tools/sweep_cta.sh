# CTA size / workers sweep for small instances
for cfg in j30 j60; do
for tw in "512 2" "256 4" "128 8"; do
  set -- $tw
  timeout 300 python bench.py --config $cfg --instances 148 --threads $1 --workers $2 --steps 2 --warmup 3 --no-cpu-baseline --no-quality --e2e-steps 0 > gpurun_out/sc.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/sc.log').read().strip().splitlines()[-1]); print('$cfg threads $1 workers $2', round(d['value']/1e6,2), 'ms/step', round(d['ms_per_step']))" || tail -2 gpurun_out/sc.log
done; done
