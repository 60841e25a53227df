#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/probe.py cfg1 50 > gpurun_out/probe_cfg1.log 2>&1
timeout 300 python tools/probe.py cfg3 4 > gpurun_out/probe_cfg3.log 2>&1
