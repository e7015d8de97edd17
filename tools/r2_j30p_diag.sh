# round 2: j30p TIME throughput regression hunt (current vs the 9a3fcb9 tree,
# sized profiles on/off)
mkdir -p gpurun_out/diag
B2="--steps 2 --warmup 1 --no-cpu-baseline --no-quality --e2e-steps 0 --no-per-config --mode time"
sum() { python -c "
import json,sys
d=json.loads(open('$1').read().strip().splitlines()[-1]); r=d['run']; print('$2', round(d['value']/1e6,2), 'M/s', 'ms', round(d['ms_per_step'],2), 'evals', r['evaluations_per_step'], 'iters', r['iterations_per_step'], 'cpm', round(r['cpm_dev'],2))
" | tee -a gpurun_out/diag/summary.txt; }
for cfg in j30p j30; do
  timeout 300 python bench.py --config $cfg --instances 148 --workers 8 --iters 1000 $B2 > gpurun_out/diag/cur_$cfg.log 2>&1; sum gpurun_out/diag/cur_$cfg.log "cur $cfg"
  timeout 300 python bench.py --config $cfg --instances 148 --workers 8 --iters 1000 $B2 --profile-slots 0 > gpurun_out/diag/cur0_$cfg.log 2>&1; sum gpurun_out/diag/cur0_$cfg.log "cur slots0 $cfg"
  (cd abl/old_tree && timeout 300 python bench.py --config $cfg --instances 148 --workers 8 --iters 1000 $B2 > ../../gpurun_out/diag/old_$cfg.log 2>&1); sum gpurun_out/diag/old_$cfg.log "old $cfg"
done
