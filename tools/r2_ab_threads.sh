# round 2: k_solve launch bounds: TIME 576 (18 warps, 56 regs) vs 640 (20 warps,
# 48 regs); CAPACITY 512 vs 576
mkdir -p gpurun_out/ab12
for cfg in "--config j120p --mode time --instances 600 --iters 1000" "--config j60p --mode time --instances 148 --workers 8 --iters 1000" "--config act300 --mode time --instances 148 --workers 2 --iters 100"; do
  bash tools/ab_args.sh 2 "$cfg" abl/t576.so abl/t640.so 2>&1 | tee -a gpurun_out/ab12/ab.txt
done
for cfg in "--config j120p --mode capacity --instances 600 --iters 300" "--config act300 --mode capacity --instances 148 --workers 2 --iters 60"; do
  bash tools/ab_args.sh 2 "$cfg" abl/t576.so abl/c576.so 2>&1 | tee -a gpurun_out/ab12/ab.txt
done
