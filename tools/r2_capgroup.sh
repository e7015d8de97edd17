# round 2: CAPACITY group 1 (thread per schedule) vs 32 (warp, rows <= 32 in
# registers) on the configs pick_cap_group sends to group 1
mkdir -p gpurun_out/cg
for cfg in "--config j120 --instances 600 --workers 2 --iters 300" "--config j60 --instances 148 --workers 8 --iters 600" "--config j30 --instances 148 --workers 8 --iters 600" "--config j30p --instances 148 --workers 8 --iters 600"; do
  for g in 1 32; do
    timeout 600 python bench.py $cfg --mode capacity --cap-group $g --steps 2 --warmup 1 --no-cpu-baseline --no-quality --e2e-steps 0 --no-per-config 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg g$g', round(d['value']/1e6,2), 'steps', round(d['roofline']['sgs_steps_per_schedule'],1))" | tee -a gpurun_out/cg/summary.txt
  done
done
