#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/dbg.log
for v in "ie 5,3,4 0.1" "stat1 5,3,4 0.1"; do
  echo "== $v" >> gpurun_out/dbg.log
  timeout 120 python tools/dbg_twoslab.py $v 2>&1 | tail -n 2 >> gpurun_out/dbg.log
done
timeout 900 python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
