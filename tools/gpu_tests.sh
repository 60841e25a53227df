#!/bin/bash
# GPU test suite (fast part unless SLOW=1)
mkdir -p gpurun_out
sel="gpu and not slow"; [ "${SLOW:-0}" = 1 ] && sel="gpu"
timeout 2400 python -m pytest tests -m "$sel" -q ${PYARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
