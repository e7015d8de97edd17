# round 2: compute-sanitizer over every search-path kernel (tools/sanitize.py)
mkdir -p gpurun_out/san3
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 \
     python tools/sanitize.py > gpurun_out/san3/$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/san3/summary.txt
  tail -4 gpurun_out/san3/$tool.log | tee -a gpurun_out/san3/summary.txt
done
