#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/small.log
for c in cfg0 small cfg1 cfg4; do for v in 2 8; do echo "== $c variant $v" >> gpurun_out/small.log
THERMO_CG_VARIANT=$v timeout 300 python tools/probe.py $c 20 2>&1 | grep -E "ms/step|solve|Error|error" | tail -n 3 >> gpurun_out/small.log; done; done
