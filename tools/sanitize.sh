#!/bin/bash
# compute-sanitizer over small parity runs (logs to gpurun_out/; TAG names them)
TAG=${TAG:-rXX}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
     python tools/sanitize_run.py > gpurun_out/${TAG}_sanitize_${tool}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/${TAG}_sanitize_${tool}.log
  tail -n 4 gpurun_out/${TAG}_sanitize_${tool}.log
done
