# session 4, call a: state check at HEAD (tests, bench lines, launch list, ncu of the batched step)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/gputests.log 2>&1; echo "rc=$?" >> gpurun_out/gputests.log
timeout 900 python bench.py > gpurun_out/bench_cfg3.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg3.log
timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 > gpurun_out/bench_cfg4.log 2>&1
THERMO_CG_TRACE=3 timeout 300 python tools/probe_batched.py 5 > gpurun_out/probe_cfg4_trace.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 300 python tools/probe_batched.py 2 > gpurun_out/probe_cfg4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sbcg_step|k_pairs|k_rows|k_refsort" -s 12 -c 4 \
    -o gpurun_out/prof_cfg4_spmm python tools/probe_batched.py 2 > gpurun_out/ncu_cfg4.log 2>&1
timeout 300 python tools/probe_latency.py 50 > gpurun_out/latency_small_configs.txt 2>&1
