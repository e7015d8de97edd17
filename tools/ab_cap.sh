for cfg in j120p j120; do for v in A B; do lib=$PWD/paper_1711_04556_b200/_lib/ab_base.so; [ $v = B ] && lib=$PWD/paper_1711_04556_b200/_lib/libb200tabu.so
RCPSP_B200_LIB=$lib timeout 300 python bench.py --config $cfg --mode capacity --instances 148 --iters 200 --steps 2 --warmup 1 --no-cpu-baseline --no-quality --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg cap $v', round(d['value']/1e6,2))"
done; done
