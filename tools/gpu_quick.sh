#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
rm -f gpurun_out/probe_all.log
for c in cfg0 cfg1 cfg2 cfg4; do timeout 300 python tools/probe.py $c 20 >> gpurun_out/probe_all.log 2>&1; done
timeout 300 python tools/probe.py cfg3 10 >> gpurun_out/probe_all.log 2>&1
