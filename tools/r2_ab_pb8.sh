# round 2: TIME phase B with one loop test per eight positions vs four
mkdir -p gpurun_out/ab17
RCPSP_B200_LIB=abl/pb8.so timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py -k "neighbourhood or orchestrate" > gpurun_out/ab17/tests.log 2>&1
tail -1 gpurun_out/ab17/tests.log
for cfg in "--config j120p --mode time --instances 600 --iters 1000" "--config j60p --mode time --instances 148 --workers 8 --iters 1000" "--config act300 --mode time --instances 148 --workers 2 --iters 100"; do
  bash tools/ab_args.sh 3 "$cfg" abl/pb4.so abl/pb8.so 2>&1 | tee -a gpurun_out/ab17/ab.txt
done
