#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck over tests/diag/sanitize_runs.py
mkdir -p gpurun_out/sanitizer
python tests/diag/sanitize_runs.py > gpurun_out/sanitizer/plain.txt 2>&1; echo "exit=$?" >> gpurun_out/sanitizer/plain.txt
for t in racecheck synccheck memcheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 50 python tests/diag/sanitize_runs.py > gpurun_out/sanitizer/$t.txt 2>&1
  echo "exit=$?" >> gpurun_out/sanitizer/$t.txt
done
