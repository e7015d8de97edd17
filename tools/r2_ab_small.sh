# round 2: small-CTA instantiations (128 x 8 / 256 x 4 launch bounds, 64
# registers) for projects of <= 64 activities vs the two-CTA bound (56)
mkdir -p gpurun_out/ab16
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py -k "orchestrate or batch_solve or multi_worker or cluster or neighbourhood" > gpurun_out/ab16/tests.log 2>&1
tail -2 gpurun_out/ab16/tests.log
for cfg in "--config j30p --mode time --instances 148 --workers 8 --iters 1000" "--config j60p --mode time --instances 148 --workers 8 --iters 1000" "--config j30 --mode time --instances 148 --workers 8 --iters 1000" "--config j60p --mode capacity --instances 148 --workers 8 --iters 600" "--config j30p --mode capacity --instances 148 --workers 8 --iters 600"; do
  bash tools/ab_args.sh 3 "$cfg" abl/nosmall.so abl/small.so 2>&1 | tee -a gpurun_out/ab16/ab.txt
done
