#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/probe_fused.log
for c in cfg0 cfg1 cfg3 cfg4; do for f in 1 0; do
echo "== $c fused $f" >> gpurun_out/probe_fused.log
THERMO_IFACE_FUSED=$f timeout 300 python tools/probe.py $c 10 2>&1 | grep -E "ms/step|iface" >> gpurun_out/probe_fused.log
done; done
THERMO_IFACE_FUSED=1 timeout 300 python tools/probe_sdc.py cfg1 mrsdc 3 2 1 20 >> gpurun_out/probe_fused.log 2>&1
