#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/probe.py cfg4 3 > gpurun_out/probe_cfg4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cgb_step" -s 2 -c 1 -o gpurun_out/prof_cfg4_win python tools/probe.py cfg4 3 > gpurun_out/ncu_cfg4.log 2>&1
