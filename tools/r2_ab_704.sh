mkdir -p gpurun_out/ab15
bash tools/ab_args.sh 3 "--config j120p --mode time --instances 600 --iters 1000" abl/l640.so abl/l704.so 2>&1 | tee -a gpurun_out/ab15/ab.txt
