mkdir -p gpurun_out/ab3
L="abl/libW.so abl/libN.so"
bash tools/ab_args.sh 2 "--config act300 --mode time --instances 148 --workers 2 --iters 100" $L | tee gpurun_out/ab3/wide.txt
bash tools/ab_args.sh 2 "--config act300 --mode capacity --instances 148 --workers 2 --iters 100" $L | tee -a gpurun_out/ab3/wide.txt
bash tools/ab_args.sh 1 "--config act300 --mode time --instances 148 --workers 1 --iters 200" $L | tee -a gpurun_out/ab3/wide.txt
bash tools/ab_args.sh 1 "--config j120p --mode time --instances 600 --workers 2" $L | tee -a gpurun_out/ab3/wide.txt
bash tools/ab_args.sh 1 "--config j120p --mode capacity --instances 600 --workers 2" $L | tee -a gpurun_out/ab3/wide.txt

