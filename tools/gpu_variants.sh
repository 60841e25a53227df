#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in 1 2 3 4 5 6 7; do
  THERMO_CG_VARIANT=$v timeout 300 python tools/probe.py cfg3 4 > gpurun_out/probe_cfg3_v$v.log 2>&1
done
THERMO_CG_VARIANT=2 timeout 300 python tools/probe.py cfg1 50 > gpurun_out/probe_cfg1_v2.log 2>&1
