#!/bin/bash
# Round-2 measurements for profiles/r02 (run through gpurun on one B200):
# bench lines (cfg3 default, cfg4), the ncu launch list of the bench command, one ncu --set full
# capture of the CG kernel (cfg3, first timed launch of the probe) and of one batched cfg4 step,
# per-config probe, latency probe, reorder probe, stationary probe.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_cfg3.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg3.log
timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 > gpurun_out/bench_cfg4.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 300 python tools/probe.py cfg3 4 > gpurun_out/probe_cfg3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cg_step -s 3 -c 1 \
    -o gpurun_out/prof_cg_cfg3 python tools/probe.py cfg3 4 > gpurun_out/ncu_cfg3.log 2>&1
timeout 300 python tools/probe_batched.py 2 > gpurun_out/probe_cfg4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cgb_step|k_pairs|k_rows" -s 9 -c 3 \
    -o gpurun_out/prof_cfg4 python tools/probe_batched.py 2 > gpurun_out/ncu_cfg4.log 2>&1
for c in cfg0 cfg1 cfg2 cfg3; do timeout 300 python tools/probe.py $c 20 2>&1 | grep -v "^\[thermo"; done > gpurun_out/probe_all_configs.txt
timeout 300 python tools/probe_batched.py 10 >> gpurun_out/probe_all_configs.txt 2>&1
timeout 300 python tools/probe_latency.py 50 > gpurun_out/latency_small_configs.txt 2>&1
timeout 300 python tools/probe_reorder.py cfg2 cfg3 10 > gpurun_out/reorder_probe.txt 2>&1
timeout 600 python tools/probe_stationary.py cfg2 > gpurun_out/stationary_probe.txt 2>&1
timeout 900 python tools/probe_stationary.py cfg3 >> gpurun_out/stationary_probe.txt 2>&1
