# the N > 1 bench path on one GPU (ranks share it; gloo plumbing): peer and epochs exchange
mkdir -p gpurun_out/mb2
for x in peer epochs; do
  BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29710 bench.py --gpus 2 --steps 3 --warmup 3 --exchange $x --instances 148 > gpurun_out/mb2/bench_2rank_$x.log 2>&1
  grep "^{" gpurun_out/mb2/bench_2rank_$x.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$x', d['value']/1e6, d['run']['parallelism'][:60], d['run'].get('peer_counters_last_step'), d['run']['cpm_dev'])" | tee -a gpurun_out/mb2/summary.txt
done
