#!/bin/bash
mkdir -p gpurun_out
for v in 1 2; do
THERMO_CG_VARIANT=$v timeout 300 python tools/probe.py cfg3 4 > gpurun_out/probe_cfg3_v$v.log 2>&1 && \
THERMO_CG_VARIANT=$v timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cg_step -s 3 -c 1 -o gpurun_out/prof_cg_cfg3_v$v python tools/probe.py cfg3 4 > gpurun_out/ncu_cfg3_v$v.log 2>&1
done
