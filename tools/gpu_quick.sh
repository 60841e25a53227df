#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/probe_ctas.log
for g in 148 96 74 48 32; do
echo "== ctas $g" >> gpurun_out/probe_ctas.log
THERMO_CG_CTAS=$g THERMO_CG_TRACE=1 timeout 300 python tools/probe.py cfg1 30 2>&1 | grep -E "trace|solve" | tail -n 2 >> gpurun_out/probe_ctas.log
done
for g in 148 74; do
echo "== cfg0 ctas $g" >> gpurun_out/probe_ctas.log
THERMO_CG_CTAS=$g THERMO_CG_TRACE=1 timeout 300 python tools/probe.py cfg0 30 2>&1 | grep -E "trace|solve" | tail -n 2 >> gpurun_out/probe_ctas.log
done
