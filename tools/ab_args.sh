# A/B/C... of library builds on the same box, interleaved, with bench args:
# tools/ab_args.sh <rounds> "<bench args>" <lib1.so> <lib2.so> ...
R=$1; ARGS=$2; shift 2
for r in $(seq $R); do
  for lib in "$@"; do
    RCPSP_B200_LIB=$lib timeout 600 python bench.py $ARGS --steps 2 --warmup 1 --no-cpu-baseline --no-quality --e2e-steps 0 --no-per-config 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $lib)', '$ARGS', round(d['value']/1e6,2), 'steps', round(d['roofline']['sgs_steps_per_schedule'],1))"
  done
done
