# populations sharing one GPU (gloo plumbing) and the cost of epoch drains at N = 1
mkdir -p gpurun_out/pop
T="python -m torch.distributed.run --nnodes 1 --master-addr 127.0.0.1"
P=29600
run() { P=$((P+1)); timeout 900 $T --nproc-per-node $1 --master-port $P tools/populations.py ${@:2} 2>>gpurun_out/pop/err.log | tail -1 | tee -a gpurun_out/pop/populations.jsonl; }
run 1 --exchange none
run 1 --exchange epochs --epochs 2
run 1 --exchange epochs --epochs 4
run 1 --exchange epochs --epochs 8
run 2 --exchange none
run 2 --exchange peer
run 2 --exchange epochs --epochs 4
run 4 --exchange none
run 4 --exchange peer
run 4 --exchange epochs --epochs 4
