#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/probe.py cfg4 3 > gpurun_out/probe_cfg4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pairs|k_rows|k_cgb_step" -s 12 -c 4 -o gpurun_out/prof_cfg4 python tools/probe.py cfg4 3 > gpurun_out/ncu_cfg4.log 2>&1
