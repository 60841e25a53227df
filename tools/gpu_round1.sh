#!/bin/bash
# first GPU call: smoke, gpu tests (not slow), probes
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/probe.py cfg1 100 > gpurun_out/probe_cfg1.log 2>&1; echo "rc=$?" >> gpurun_out/probe_cfg1.log
timeout 600 python tools/probe.py cfg3 10 > gpurun_out/probe_cfg3.log 2>&1; echo "rc=$?" >> gpurun_out/probe_cfg3.log
nproc > gpurun_out/host.txt; lscpu | head -20 >> gpurun_out/host.txt; free -g >> gpurun_out/host.txt
