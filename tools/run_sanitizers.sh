#!/bin/bash
# compute-sanitizer over tools/sanitize_smoke.py (every kernel, smoke size);
# logs -> gpurun_out/sanitizer/<tool>.log
mkdir -p gpurun_out/sanitizer
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 300 python tools/sanitize_smoke.py > gpurun_out/sanitizer/plain.log 2>&1; echo "plain rc=$?"
for tool in memcheck synccheck racecheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  timeout ${SAN_TIMEOUT:-900} $CS --tool $tool $extra --target-processes all --print-limit 200 \
     python tools/sanitize_smoke.py $SAN_ONLY > gpurun_out/sanitizer/$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitizer/$tool.log
done
