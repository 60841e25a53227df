#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/probe.py cfg4 3 > gpurun_out/probe_cfg4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cgb_step|k_pairs|k_rows" -s 6 -c 3 -o gpurun_out/prof_cfg4_final python tools/probe.py cfg4 3 > gpurun_out/ncu_cfg4.log 2>&1
