#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/probe.py cfg1 50 > gpurun_out/probe_cfg1.log 2>&1
timeout 300 python tools/probe.py cfg3 4 > gpurun_out/probe_cfg3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cg_step -s 3 -c 1 -o gpurun_out/prof_cg_cfg3 python tools/probe.py cfg3 4 > gpurun_out/ncu_cfg3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_pairs|k_rows" -s 9 -c 3 -o gpurun_out/prof_iface_cfg3 python tools/probe.py cfg3 4 > gpurun_out/ncu_iface.log 2>&1
