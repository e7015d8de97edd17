# round 2: TIME k_solve instantiated twice -- 640-thread launch bound (48
# registers) for projects above 64 activities, 576 otherwise -- vs HEAD
mkdir -p gpurun_out/ab14
timeout 1200 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_long.py tests/test_gpu_parity.py -k "long or orchestrate or neighbourhood or batch_solve or cluster or sized or multi_worker" > gpurun_out/ab14/tests.log 2>&1
tail -2 gpurun_out/ab14/tests.log
for cfg in "--config j120p --mode time --instances 600 --iters 1000" "--config j120 --mode time --instances 600 --iters 1000" "--config j60p --mode time --instances 148 --workers 8 --iters 1000" "--config act300 --mode time --instances 148 --workers 2 --iters 100"; do
  bash tools/ab_args.sh 3 "$cfg" abl/head3.so abl/lb.so 2>&1 | tee -a gpurun_out/ab14/ab.txt
done
