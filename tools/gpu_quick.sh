#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_fullrun.py -m gpu -x -q -k "batched or cfg4" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/probe_exp.log
THERMO_CG_TRACE=1 timeout 300 python tools/probe.py cfg4 5 2>&1 | grep -E "trace|ms/step|solve" | tail -n 3 >> gpurun_out/probe_exp.log
