# round 2: phase B per eight positions in the large-project kernel only (compile-time)
mkdir -p gpurun_out/ab19
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_long.py -k "neighbourhood or orchestrate or long or sized or cluster or batch_solve" > gpurun_out/ab19/tests.log 2>&1
tail -1 gpurun_out/ab19/tests.log
for cfg in "--config j120p --mode time --instances 600 --iters 1000" "--config j60p --mode time --instances 148 --workers 8 --iters 1000" "--config act300 --mode time --instances 148 --workers 2 --iters 100" "--config j120 --mode time --instances 600 --iters 1000"; do
  bash tools/ab_args.sh 3 "$cfg" abl/pb4.so abl/long8k.so 2>&1 | tee -a gpurun_out/ab19/ab.txt
done
