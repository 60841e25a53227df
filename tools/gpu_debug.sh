#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/debug6.log
for d in 4 5 6 7; do
  echo "== debug $d" >> gpurun_out/debug6.log
  THERMO_CG_DEBUG=$d THERMO_CG_TRACE=1 timeout 300 python tools/probe.py cfg3 2 2>&1 | grep -E "trace" >> gpurun_out/debug6.log
done
