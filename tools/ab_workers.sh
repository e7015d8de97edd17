for r in 1 2 3; do for w in 2 4; do
timeout 300 python bench.py --workers $w --steps 3 --warmup 2 --no-cpu-baseline --no-quality --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('workers $w', round(d['value']/1e6,2), 'cpm', round(d['config']['cpm_dev'],3))"
done; done
