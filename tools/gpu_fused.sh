#!/bin/bash
# fused (one barrier per iteration) vs two-phase CG kernels: tests, then probes per config
mkdir -p gpurun_out
rm -f gpurun_out/fused.log
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x -k "variant or fused or parity" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log >> gpurun_out/fused.log
for c in cfg1 cfg2 cfg3; do for v in 2 8 4 9; do echo "== $c variant $v" >> gpurun_out/fused.log
THERMO_CG_VARIANT=$v THERMO_CG_VERBOSE=1 timeout 300 python tools/probe.py $c 10 2>&1 | grep -E "thermo cg|ms/step|solve|Error|error" | tail -n 4 >> gpurun_out/fused.log; done; done
