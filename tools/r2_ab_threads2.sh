# round 2: launch bounds, second pass on the small projects
mkdir -p gpurun_out/ab13
for cfg in "--config j60p --mode capacity --instances 148 --workers 8 --iters 600" "--config j30p --mode capacity --instances 148 --workers 8 --iters 600" "--config j120 --mode capacity --instances 600 --iters 300"; do
  bash tools/ab_args.sh 3 "$cfg" abl/t576.so abl/c576.so 2>&1 | tee -a gpurun_out/ab13/ab.txt
done
for cfg in "--config j60p --mode time --instances 148 --workers 8 --iters 1000" "--config j30p --mode time --instances 148 --workers 8 --iters 1000"; do
  bash tools/ab_args.sh 3 "$cfg" abl/t576.so abl/t640.so 2>&1 | tee -a gpurun_out/ab13/ab.txt
done
