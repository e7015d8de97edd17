# round 2: compute-sanitizer after the CAPACITY register-row / launch-bound
# changes: memcheck over every section, racecheck (error level) per section
out=gpurun_out/san4
mkdir -p $out
timeout 1500 compute-sanitizer --tool memcheck --print-limit 50 --error-exitcode 9 python tools/sanitize.py > $out/memcheck.log 2>&1
echo "memcheck rc=$? $(tail -1 $out/memcheck.log)" | tee -a $out/summary.txt
for sec in K1 misc K2 K3 K4; do
  timeout 900 compute-sanitizer --tool racecheck --racecheck-detect-level error \
     --print-limit 100 --error-exitcode 9 python tools/sanitize.py $sec > $out/race_$sec.log 2>&1
  echo "racecheck $sec rc=$? $(grep 'RACECHECK SUMMARY' $out/race_$sec.log)" | tee -a $out/summary.txt
done
timeout 900 compute-sanitizer --tool synccheck --print-limit 50 --error-exitcode 9 python tools/sanitize.py K1 K2 K3 > $out/synccheck.log 2>&1
echo "synccheck rc=$? $(tail -1 $out/synccheck.log)" | tee -a $out/summary.txt
