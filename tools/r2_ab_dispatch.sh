# round 2: evaluator dispatch inlined (cur) vs noinline (dni) in the search kernel
mkdir -p gpurun_out/ab7
for cfg in "--config j30 --mode time --instances 148 --workers 8 --iters 1000" "--config j30p --mode time --instances 148 --workers 8 --iters 1000" "--config j60p --mode time --instances 148 --workers 8 --iters 1000" "--config j120p --mode time --instances 600 --iters 1000" "--config j120p --mode capacity --instances 600 --iters 300"; do
  bash tools/ab_args.sh 3 "$cfg" abl/cur.so abl/dni.so 2>&1 | tee -a gpurun_out/ab7/ab.txt
done
