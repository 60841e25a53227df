#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -q -k "consumer_groups or variants" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/variants3.log
for v in 3 5; do echo "== cfg3 variant $v" >> gpurun_out/variants3.log
THERMO_CG_VARIANT=$v THERMO_CG_VERBOSE=1 THERMO_CG_TRACE=1 timeout 300 python tools/probe.py cfg3 6 2>&1 | grep -E "thermo|ms/step|Error|error" | tail -n 4 >> gpurun_out/variants3.log; done
