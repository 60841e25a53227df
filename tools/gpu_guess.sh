#!/bin/bash
# CG initial guess (0 = T^n, 1 linear, 2 quadratic) and ring budget on cfg2/cfg3
mkdir -p gpurun_out
rm -f gpurun_out/guess.log
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log >> gpurun_out/guess.log
for c in cfg2 cfg3; do for g in 0 1 2; do for kb in 210 224; do
[ "$c" = cfg2 ] && [ "$kb" = 210 ] && continue
echo "== $c guess $g smem ${kb}KB" >> gpurun_out/guess.log
GUESS=$g THERMO_CG_SMEM_KB=$kb THERMO_CG_VERBOSE=1 THERMO_CG_TRACE=1 timeout 300 python tools/probe.py $c 10 2>&1 | grep -E "thermo|ms/step|solve|iterations|Error|error" | tail -n 6 >> gpurun_out/guess.log; done; done; done
