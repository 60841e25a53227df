#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/probe_cfg4_v.log
THERMO_CGB_CR=4 timeout 900 python -m pytest tests/test_gpu_batched.py -m gpu -x -q -k "not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for v in "8 3" "8 2" "4 8" "4 4" "4 3" "16 2"; do set -- $v
echo "== CR $1 NS $2" >> gpurun_out/probe_cfg4_v.log
THERMO_CGB_CR=$1 THERMO_CGB_NS=$2 THERMO_CG_TRACE=1 timeout 300 python tools/probe.py cfg4 3 2>&1 | grep -E "thermo|solve" >> gpurun_out/probe_cfg4_v.log
done
