#!/bin/bash
# compute-sanitizer over small runs of every CUDA path (tools/sanitize.py)
mkdir -p gpurun_out
python tools/sanitize.py > gpurun_out/sanitize_plain.log 2>&1
for tool in memcheck synccheck racecheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
