# round 2: search-loop pieces out of line: v1 = evaluator dispatch noinline,
# v2 + filter, v3 + the whole evaluation phase, v4 both
mkdir -p gpurun_out/ab8
for cfg in "--config j30 --mode time --instances 148 --workers 8 --iters 1000" "--config j30p --mode time --instances 148 --workers 8 --iters 1000" "--config j60p --mode time --instances 148 --workers 8 --iters 1000" "--config j120p --mode time --instances 600 --iters 1000"; do
  bash tools/ab_args.sh 2 "$cfg" abl/v1.so abl/v2.so abl/v3.so abl/v4.so 2>&1 | tee -a gpurun_out/ab8/ab.txt
done
