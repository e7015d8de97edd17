# round 2: compute-sanitizer on the large-project search kernel (K3L section)
out=gpurun_out/san5
mkdir -p $out
timeout 1500 compute-sanitizer --tool memcheck --print-limit 50 --error-exitcode 9 python tools/sanitize.py K3L > $out/memcheck.log 2>&1
echo "memcheck rc=$? $(tail -1 $out/memcheck.log)" | tee -a $out/summary.txt
timeout 1500 compute-sanitizer --tool racecheck --racecheck-detect-level error --print-limit 100 --error-exitcode 9 python tools/sanitize.py K3L > $out/racecheck.log 2>&1
echo "racecheck rc=$? $(grep 'RACECHECK SUMMARY' $out/racecheck.log)" | tee -a $out/summary.txt
timeout 1500 compute-sanitizer --tool synccheck --print-limit 50 --error-exitcode 9 python tools/sanitize.py K3L > $out/synccheck.log 2>&1
echo "synccheck rc=$? $(tail -1 $out/synccheck.log)" | tee -a $out/summary.txt
grep -h "K3L ok" $out/*.log | head -1
