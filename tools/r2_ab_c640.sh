mkdir -p gpurun_out/ab20
for cfg in "--config j120p --mode capacity --instances 600 --iters 300" "--config j60p --mode capacity --instances 148 --workers 8 --iters 600" "--config j120 --mode capacity --instances 600 --iters 300"; do
  bash tools/ab_args.sh 3 "$cfg" abl/c576b.so abl/c640.so 2>&1 | tee -a gpurun_out/ab20/ab.txt
done
