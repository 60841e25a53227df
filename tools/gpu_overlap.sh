#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/overlap.log
for c in cfg0 small medium cfg1; do for o in "0 24" "1 16" "1 24" "1 32"; do set -- $o
echo "== $c overlap $1 free SMs $2" >> gpurun_out/overlap.log
THERMO_OVERLAP=$1 THERMO_OVERLAP_SMS=$2 timeout 300 python tools/probe.py $c 20 2>&1 | grep -E "ms/step|solve|Error|error" | tail -n 3 >> gpurun_out/overlap.log; done; done
