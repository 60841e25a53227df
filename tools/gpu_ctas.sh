#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/ctas.log
for c in cfg0 small medium cfg1; do for g in 148 74 37 16 4 1; do echo "== $c ctas $g" >> gpurun_out/ctas.log
THERMO_CG_CTAS=$g THERMO_CG_TRACE=1 timeout 300 python tools/probe.py $c 20 2>&1 | grep -E "thermo trace|ms/step|Error|error" | tail -n 2 >> gpurun_out/ctas.log; done; done
