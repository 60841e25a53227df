#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in 0 1 2; do
  THERMO_CG_VARIANT=$v timeout 300 python tools/probe.py cfg3 4 > gpurun_out/probe_cfg3_v$v.log 2>&1
  THERMO_CG_VARIANT=$v timeout 300 python tools/probe.py cfg1 50 > gpurun_out/probe_cfg1_v$v.log 2>&1
done
