# A/B on both workloads: tools/ab_bench2.sh <libA.so> <libB.so> [rounds]
A=$1; B=$2; R=${3:-2}
for cfg in j120p j120; do
for r in $(seq $R); do
  for v in A B; do
    lib=$A; [ $v = B ] && lib=$B
    RCPSP_B200_LIB=$lib timeout 300 python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline --no-quality --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg $v', round(d['value']/1e6,2))"
  done
done; done
