# workers-per-instance sweep on the default workload (600 Gen-P j120 instances)
for w in 2 3 4; do
  timeout 300 python bench.py --workers $w --steps 2 --warmup 2 --no-cpu-baseline --no-quality --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('workers $w', round(d['value']/1e6,2), 'ms/step', round(d['ms_per_step']), 'cpm', round(d['config']['cpm_dev'],2))"
done
