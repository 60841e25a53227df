#!/bin/bash
# Round 2, session 4: the gpurun command lines behind this session's files under profiles/r02/
# (one B200; every step under its own timeout so that a hang cannot eat the GPU budget).
#   bash tools/gpu_r2_session4.sh final     full -m gpu suite, smoke, bench lines (cfg3, cfg4), launch list, ncu captures
#   bash tools/gpu_r2_session4.sh latency   small configurations: resident / cluster / streaming kernels, traces
#   bash tools/gpu_r2_session4.sh ahead     configs 2 and 3 with and without the ahead mode
#   bash tools/gpu_r2_session4.sh e2e       batched end-to-end probe
mkdir -p gpurun_out
case "$1" in
final)
    timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 --durations=8 > gpurun_out/gputests.log 2>&1; echo "rc=$?" >> gpurun_out/gputests.log
    timeout 200 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
    timeout 900 python bench.py > gpurun_out/bench_cfg3.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg3.log
    timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 > gpurun_out/bench_cfg4.log 2>&1
    timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv \
        python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
    timeout 300 python tools/probe.py cfg3 4 > gpurun_out/probe_cfg3.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cg_step -s 3 -c 1 \
        -o gpurun_out/prof_cg_cfg3 python tools/probe.py cfg3 4 > gpurun_out/ncu_cfg3.log 2>&1
    timeout 300 python tools/probe_batched.py 2 > gpurun_out/probe_cfg4.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sbcg_step|k_pairs|k_rows|k_refsort" -s 12 -c 4 \
        -o gpurun_out/prof_cfg4_spmm python tools/probe_batched.py 2 > gpurun_out/ncu_cfg4.log 2>&1
    timeout 200 python tools/probe.py medium 20 > gpurun_out/probe_medium.log 2>&1 && \
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_cg_resident|k_pairs|k_rows|k_refsort" -s 20 -c 6 \
        -o gpurun_out/prof_resident_medium python tools/probe.py medium 20 > gpurun_out/ncu_resident.log 2>&1
    for c in cfg0 cfg1 cfg2 cfg3; do timeout 300 python tools/probe.py $c 20 2>&1 | grep -v "^\[thermo"; done > gpurun_out/probe_all_configs.txt
    timeout 300 python tools/probe_batched.py 10 >> gpurun_out/probe_all_configs.txt 2>&1
    ;;
latency)
    timeout 300 python tools/probe_latency.py 50 > gpurun_out/latency_small_configs.txt 2>&1
    for c in cfg0 medium; do THERMO_CG_TRACE=1 timeout 120 python tools/probe.py $c 20 2>&1 | grep -v "^\[thermo c" | tail -4; done >> gpurun_out/latency_small_configs.txt
    ;;
ahead)
    out=gpurun_out/ahead_large.txt; : > $out
    for c in cfg2 cfg3; do for a in 16 0; do echo "== $c THERMO_AHEAD=$a" >> $out; THERMO_AHEAD=$a timeout 300 python tools/probe.py $c 20 2>&1 | grep -v "^\[thermo cg\]" | tail -4 >> $out; done; done
    ;;
e2e)
    timeout 600 python tools/probe_e2e.py 20 > gpurun_out/probe_e2e_cfg4.txt 2>&1
    ;;
*) echo "usage: $0 final|latency|ahead|e2e"; exit 2 ;;
esac
