#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/probe_exp.log
THERMO_CG_TRACE=1 timeout 300 python tools/probe.py cfg4 5 2>&1 | grep -E "trace|ms/step|solve" | tail -n 3 >> gpurun_out/probe_exp.log
