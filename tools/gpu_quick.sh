#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/work_precision_batched.py 64 60 > gpurun_out/work_precision_batched.txt 2>&1
