#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batched.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/probe_order.log
for o in 1 0; do
echo "== order $o" >> gpurun_out/probe_order.log
THERMO_CGB_ORDER=$o THERMO_CG_TRACE=1 timeout 300 python tools/probe.py cfg4 5 2>&1 | grep -E "trace|solve" >> gpurun_out/probe_order.log
done
