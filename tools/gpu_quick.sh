#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/probe_exp.log
for mb in 1 2; do echo "== minb $mb" >> gpurun_out/probe_exp.log
THERMO_CGB_MINB=$mb THERMO_CG_TRACE=1 timeout 300 python tools/probe.py cfg4 5 2>&1 | grep -E "trace|solve" | tail -n 2 >> gpurun_out/probe_exp.log; done
THERMO_CGB_MINB=2 timeout 900 python -m pytest tests/test_gpu_batched.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
