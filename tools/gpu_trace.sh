#!/bin/bash
mkdir -p gpurun_out
for v in 0 1 2 3; do
  THERMO_CG_TRACE=1 THERMO_CG_VARIANT=$v timeout 300 python tools/probe.py cfg3 2 > gpurun_out/trace_cfg3_v$v.log 2>&1
done
