# GPU tests (fine-grained exchange) + ncu of the CAP evaluator (register path) + sweep
mkdir -p gpurun_out/p3
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/p3/gpu_tests.log 2>&1
tail -3 gpurun_out/p3/gpu_tests.log
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-quality --e2e-steps 0 --no-per-config"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -c 1 -o gpurun_out/p3/cap_j120p $B --config j120p --mode capacity --instances 148 --iters 100 > gpurun_out/p3/ncu_cap_j120p.log 2>&1
python tools/ncu_summary.py gpurun_out/p3/cap_j120p.ncu-rep > gpurun_out/p3/cap_j120p.txt 2>&1
python tools/ncu_lines.py gpurun_out/p3/cap_j120p.ncu-rep 80 > gpurun_out/p3/cap_j120p_lines.txt 2>&1
ncu -i gpurun_out/p3/cap_j120p.ncu-rep --page source --csv --print-source sass > gpurun_out/p3/cap_j120p_sass.csv 2>/dev/null
B2="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-quality --e2e-steps 0 --no-per-config"
for c in "j120p 600 2 1000 capacity" "j30p 148 8 1000 time" "j60p 148 8 1000 time" "j120p 600 2 1000 time"; do
  set -- $c
  timeout 600 $B2 --config $1 --instances $2 --workers $3 --iters $4 --mode $5 > gpurun_out/p3/b_$1_$5.log 2>&1
  python -c "
import json
try:
  d=json.loads(open('gpurun_out/p3/b_$1_$5.log').read().strip().splitlines()[-1]); print('$1 $5', round(d['value']/1e6,2), 'M/s frac', round(d['roofline']['frac'],4), 'steps/sched', round(d['roofline']['sgs_steps_per_schedule'],1), 'cpm', round(d['run']['cpm_dev'],2))
except Exception as e: print('$1 $5 FAILED', open('gpurun_out/p3/b_$1_$5.log').read()[-600:])
" | tee -a gpurun_out/p3/summary.txt
done
