#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/probe_exp.log
for pt in 1 0; do for c in cfg1 cfg3; do echo "== $c pattern $pt" >> gpurun_out/probe_exp.log
THERMO_CG_PATTERN=$pt THERMO_CG_TRACE=1 timeout 300 python tools/probe.py $c 10 2>&1 | grep -E "trace|N=|ms/step|solve" | tail -n 4 >> gpurun_out/probe_exp.log; done; done
