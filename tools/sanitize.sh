#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py: memcheck, racecheck, synccheck (GPU box).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for case in cfg1 edge norm mask tp1; do
    echo "== $tool $case"
    timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 20 \
      python tools/sanitize_cases.py $case 2>&1 | tail -8
    echo "rc=${PIPESTATUS[0]}"
  done
done
