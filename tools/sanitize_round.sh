#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck over tools/sanitize_driver.py.
# Usage (under gpurun): bash tools/sanitize_round.sh <tag>
tag=${1:-r2}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 100000 \
      python tools/sanitize_driver.py > gpurun_out/${tag}_sanitize_${tool}.log 2>&1
  echo "$tool rc $?"; tail -3 gpurun_out/${tag}_sanitize_${tool}.log
done
