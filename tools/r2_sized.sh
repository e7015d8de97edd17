mkdir -p gpurun_out/sz
timeout 1200 python -m pytest tests/test_gpu_parity.py -k "sized or neighbourhood or orchestrate or cluster or full_sgs" tests/test_gpu_long.py -q -x -p no:cacheprovider > gpurun_out/sz/tests.log 2>&1; tail -1 gpurun_out/sz/tests.log
for r in 1 2; do
for ps in "" "--profile-slots 0"; do
  timeout 600 python bench.py --config act300 --mode time --instances 148 --workers 2 --iters 100 --steps 2 --warmup 1 --no-cpu-baseline --no-quality --e2e-steps 0 --no-per-config $ps 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('act300 time [$ps]', round(d['value']/1e6,2), 'steps', round(d['roofline']['sgs_steps_per_schedule'],1))" | tee -a gpurun_out/sz/ab.txt
done
done
for ps in "" "--profile-slots 0"; do
  timeout 600 python bench.py --config j120p --mode time --instances 600 --workers 2 --steps 2 --warmup 1 --no-cpu-baseline --no-quality --e2e-steps 0 --no-per-config $ps 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('j120p time [$ps]', round(d['value']/1e6,2))" | tee -a gpurun_out/sz/ab.txt
done
