#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
THERMO_CG_TRACE=1 timeout 300 python tools/probe.py cfg4 5 > gpurun_out/probe_cfg4.log 2>&1
