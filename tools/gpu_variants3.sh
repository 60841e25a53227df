#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/variants3.log
for v in 2 3 5 6; do for kb in 210 224; do echo "== cfg3 variant $v smem $kb" >> gpurun_out/variants3.log
THERMO_CG_SMEM_KB=$kb THERMO_CG_VARIANT=$v THERMO_CG_VERBOSE=1 THERMO_CG_TRACE=1 timeout 300 python tools/probe.py cfg3 6 2>&1 | grep -E "thermo|ms/step|Error|error" | tail -n 4 >> gpurun_out/variants3.log; done; done
