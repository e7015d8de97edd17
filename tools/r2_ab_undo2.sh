mkdir -p gpurun_out/ab22
RCPSP_B200_LIB=abl/u8.so timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py -k "neighbourhood or orchestrate or large_project" > gpurun_out/ab22/tests.log 2>&1
tail -1 gpurun_out/ab22/tests.log
for cfg in "--config j120p --mode time --instances 600 --iters 1000" "--config j60p --mode time --instances 148 --workers 8 --iters 1000"; do
  bash tools/ab_args.sh 3 "$cfg" abl/head5.so abl/u8.so abl/u2.so 2>&1 | tee -a gpurun_out/ab22/ab.txt
done
