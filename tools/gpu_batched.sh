#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not cfg1_full" > gpurun_out/pytest_batched.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_batched.log
timeout 600 python tools/probe.py cfg4 10 > gpurun_out/probe_cfg4.log 2>&1
timeout 600 python tools/probe.py cfg1 50 > gpurun_out/probe_cfg1.log 2>&1
