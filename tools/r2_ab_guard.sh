# round 2: CAPACITY fast path: the r > 32 store loop behind a uniform guard
mkdir -p gpurun_out/ab11
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_state.py > gpurun_out/ab11/tests.log 2>&1
tail -2 gpurun_out/ab11/tests.log
for cfg in "--config act300 --mode capacity --instances 148 --workers 2 --iters 60" "--config j120p --mode capacity --instances 600 --iters 300" "--config j60p --mode capacity --instances 148 --workers 8 --iters 600"; do
  bash tools/ab_args.sh 3 "$cfg" abl/head.so abl/guard.so 2>&1 | tee -a gpurun_out/ab11/ab.txt
done
