#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/probe_cfg4_v.log
for pm in 1; do
echo "== pmode $pm" >> gpurun_out/probe_cfg4_v.log
THERMO_CGB_PMODE=$pm THERMO_CG_TRACE=1 timeout 300 python tools/probe.py cfg4 3 2>&1 | grep -E "trace|solve" >> gpurun_out/probe_cfg4_v.log
done
