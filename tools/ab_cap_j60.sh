for lib in "$@"; do
  RCPSP_B200_LIB=$lib timeout 300 python bench.py --config j60 --mode capacity --instances 148 --workers 8 --iters 1000 --steps 2 --warmup 2 --no-cpu-baseline --no-quality --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('j60cap $(basename $lib)', round(d['value']/1e6,2))"
done
