# A/B/C... of several library builds on the same box, interleaved:
# tools/ab_multi.sh <rounds> <config> <lib1.so> <lib2.so> ...
R=$1; CFG=$2; shift 2
for r in $(seq $R); do
  for lib in "$@"; do
    RCPSP_B200_LIB=$lib timeout 300 python bench.py --config $CFG --steps 3 --warmup 2 --no-cpu-baseline --no-quality --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$CFG $(basename $lib)', round(d['value']/1e6,2))"
  done
done
