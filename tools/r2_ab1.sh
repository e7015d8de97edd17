mkdir -p gpurun_out/ab
L="abl/libA.so abl/libB.so abl/libC.so abl/libD.so"
bash tools/ab_args.sh 2 "--config j120p --mode capacity --instances 600 --workers 2" $L | tee gpurun_out/ab/cap.txt
bash tools/ab_args.sh 1 "--config act300 --mode capacity --instances 148 --workers 2 --iters 100" $L | tee -a gpurun_out/ab/cap.txt
bash tools/ab_args.sh 1 "--config j60p --mode capacity --instances 148 --workers 8" $L | tee -a gpurun_out/ab/cap.txt
