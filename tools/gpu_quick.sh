#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/probe_exp.log
for c in cfg1 cfg3 cfg4; do timeout 300 python tools/probe.py $c 10 2>&1 | grep -E "iface" | tail -n 1 >> gpurun_out/probe_exp.log; done
