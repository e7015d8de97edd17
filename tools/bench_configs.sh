mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "neighbourhood or run_chunk or orchestrate or full_sgs" > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
for cfg in j120 j30 j60 act300; do
 for mode in time capacity; do
  it=1000; [ $cfg = act300 ] && it=300
  timeout 300 python bench.py --config $cfg --mode $mode --iters $it --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b_${cfg}_${mode}.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/b_${cfg}_${mode}.log').read().strip().splitlines()[-1]); print('$cfg $mode', round(d['value']/1e6,2), 'M/s', 'ms/step', round(d['ms_per_step']), 'cpm_dev', round(d['config']['cpm_dev'],2))" || tail -3 gpurun_out/b_${cfg}_${mode}.log
 done
done
tail -2 gpurun_out/gpu_tests.log
