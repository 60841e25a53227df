#!/bin/bash
# S-phase bound analysis on cfg3: THERMO_CG_DEBUG 1 = consumers skip row work, 2 = no window
# copies, 3 = both (timings only; results invalid, fixed 50 iterations)
mkdir -p gpurun_out
for d in 0 1 2 3; do echo "== debug $d" >> gpurun_out/dbgphase.log
THERMO_CG_DEBUG=$d THERMO_CG_TRACE=1 timeout 300 python tools/probe.py cfg3 3 2>&1 | grep -E "trace|ms/step|solve" | tail -n 3 >> gpurun_out/dbgphase.log; done
