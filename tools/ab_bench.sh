# A/B of two library builds on the same box: tools/ab_bench.sh <libA.so> <libB.so> [rounds]
# (build a variant with: make -C paper_1711_04556_b200 OUT=/abs/path/libX.so)
A=$1; B=$2; R=${3:-3}
for r in $(seq $R); do
  for v in A B; do
    lib=$A; [ $v = B ] && lib=$B
    RCPSP_B200_LIB=$lib timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-quality --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e6,2))"
  done
done
