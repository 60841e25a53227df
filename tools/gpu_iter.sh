#!/bin/bash
# iteration check: fast GPU tests, then traced probes of cfg1/cfg2/cfg3
mkdir -p gpurun_out
rm -f gpurun_out/iter.log
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log >> gpurun_out/iter.log
for c in ${CFGS:-cfg1 cfg2 cfg3}; do echo "== $c" >> gpurun_out/iter.log
THERMO_CG_VERBOSE=1 THERMO_CG_TRACE=1 timeout 300 python tools/probe.py $c ${STEPS:-5} 2>&1 | grep -E "thermo|ms/step|solve|Error|error" | tail -n 6 >> gpurun_out/iter.log; done
