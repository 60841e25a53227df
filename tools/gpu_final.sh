#!/bin/bash
# round-end refresh: full GPU suite (incl. slow full runs), full-run parity table, bench, ncu
# launch list of the bench command, ncu --set full of the CG kernel (cfg3, first timed launch of
# the probe) and of one step's interface kernels, per-config probes
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/fullrun_errors.py > gpurun_out/fullrun_parity.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 300 python tools/probe.py cfg3 4 > gpurun_out/probe_cfg3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cg_step -s 3 -c 1 -o gpurun_out/prof_cg_cfg3 python tools/probe.py cfg3 4 > gpurun_out/ncu_cfg3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_pairs|k_rows|k_extrap" -s 9 -c 4 -o gpurun_out/prof_iface_cfg3 python tools/probe.py cfg3 4 > gpurun_out/ncu_iface.log 2>&1
rm -f gpurun_out/probe_all.log
for c in cfg0 cfg1 cfg2 cfg3 cfg4; do THERMO_CG_TRACE=1 timeout 600 python tools/probe.py $c 20 >> gpurun_out/probe_all.log 2>&1; done
