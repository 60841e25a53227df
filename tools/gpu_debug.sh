#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for cfgv in "32 0" "64 0" "32 1"; do set -- $cfgv
  echo "== gap $1 prefetch $2" >> gpurun_out/debug5.log
  THERMO_CG_PREFETCH=$2 THERMO_CG_GAP=$1 THERMO_CG_TRACE=1 timeout 300 python tools/probe.py cfg3 3 2>&1 | grep -E "trace|us/iter" >> gpurun_out/debug5.log
done
THERMO_CG_TRACE=1 timeout 300 python tools/probe.py cfg1 30 2>&1 | grep -E "trace|us/iter" >> gpurun_out/debug5.log
