# compute-sanitizer over tools/gpu/sanitize_cases.py, one log per tool and case
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for case in screen exact fit knn; do
    timeout 900 $CS --tool $tool --print-limit 20 --error-exitcode 9 python tools/gpu/sanitize_cases.py $case \
      > gpurun_out/sanitize/${tool}_${case}.log 2>&1
    echo "$tool $case rc=$?" | tee -a gpurun_out/sanitize/summary.txt
  done
done
