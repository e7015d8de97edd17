for lib in "$@"; do
  for cfg in j120 j60; do
  RCPSP_B200_LIB=$lib timeout 300 python bench.py --config $cfg --mode capacity --instances $([ $cfg = j120 ] && echo 600 || echo 148) --workers $([ $cfg = j120 ] && echo 2 || echo 8) --iters 1000 --steps 2 --warmup 2 --no-cpu-baseline --no-quality --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg cap $(basename $lib)', round(d['value']/1e6,2))"
  done
done
