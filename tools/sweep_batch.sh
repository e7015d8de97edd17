for cfg in "148 2" "296 1" "600 1" "600 2" "296 2"; do
  set -- $cfg
  timeout 300 python bench.py --instances $1 --workers $2 --steps 2 --warmup 3 --no-cpu-baseline --no-quality --e2e-steps 0 > gpurun_out/sw.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]); print('inst $1 workers $2', round(d['value']/1e6,2), 'ms/step', round(d['ms_per_step']), 'cpm', round(d['config']['cpm_dev'],2))"
done
