#!/bin/bash
mkdir -p gpurun_out
python tools/probe.py cfg1 50 > gpurun_out/probe_cfg1.log 2>&1
python tools/probe.py cfg3 4 > gpurun_out/probe_cfg3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_cg_step -s 3 -c 1 -o gpurun_out/prof_cg_cfg3 python tools/probe.py cfg3 4 > gpurun_out/ncu_cfg3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 40 --csv --log-file gpurun_out/launches_cfg1.csv python tools/probe.py cfg1 50 > gpurun_out/ncu_cfg1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_iface_assemble -s 5 -c 1 -o gpurun_out/prof_iface_cfg1 python tools/probe.py cfg1 50 > gpurun_out/ncu_iface.log 2>&1
