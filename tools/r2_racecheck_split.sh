# round 2: racecheck per tools/sanitize.py section, errors only (detect level
# error), so the shared-memory hazards can be attributed to one kernel path
out=gpurun_out/race_split
mkdir -p $out
for sec in K1 misc K2 K3 sized K4; do
  timeout 900 compute-sanitizer --tool racecheck --racecheck-detect-level error \
     --print-limit 400 --error-exitcode 9 python tools/sanitize.py $sec > $out/$sec.log 2>&1
  echo "$sec rc=$? $(grep 'RACECHECK SUMMARY' $out/$sec.log)" | tee -a $out/summary.txt
  grep -A12 '^========= Error' $out/$sec.log | grep -oE 'at [^ ]+.* in [a-z_]+\.cuh?:[0-9]+' \
     | sed -E 's/\(.*\)//' | sort | uniq -c | sort -rn | head -20 | tee -a $out/summary.txt
done
