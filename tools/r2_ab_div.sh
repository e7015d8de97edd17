# round 2: diversification's serial thread-0 part done by warp 0 (prefix +
# ballot search), A/B against HEAD; diversify / trajectory tests first
mkdir -p gpurun_out/ab10
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_long.py -k "diversify or orchestrate or long or rng or sized or batch_solve" > gpurun_out/ab10/tests.log 2>&1
tail -3 gpurun_out/ab10/tests.log
for cfg in "--config j30p --mode time --instances 148 --workers 8 --iters 1000" "--config j30 --mode time --instances 148 --workers 8 --iters 1000" "--config j60p --mode time --instances 148 --workers 8 --iters 1000" "--config j120p --mode time --instances 600 --iters 1000"; do
  bash tools/ab_args.sh 3 "$cfg" abl/head.so abl/div.so 2>&1 | tee -a gpurun_out/ab10/ab.txt
done
