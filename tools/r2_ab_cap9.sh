# round 2: CAPACITY rows > 32 entries: first window from registers with
# continuation (cap_update_long) vs the i0-aligned generic form
mkdir -p gpurun_out/ab9
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_state.py "tests/test_gpu_parity.py" -k "cap or capacity or state or neighbourhood or fuzz" > gpurun_out/ab9/tests.log 2>&1
tail -3 gpurun_out/ab9/tests.log
for cfg in "--config j120p --mode capacity --instances 600 --iters 300" "--config act300 --mode capacity --instances 148 --workers 2 --iters 60" "--config j60p --mode capacity --instances 148 --workers 8 --iters 600"; do
  bash tools/ab_args.sh 3 "$cfg" abl/base2.so abl/long.so 2>&1 | tee -a gpurun_out/ab9/ab.txt
done
