mkdir -p gpurun_out
timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 > gpurun_out/bench_cfg4.log 2>&1
THERMO_CG_TRACE=3 timeout 300 python tools/probe_batched.py 5 > gpurun_out/probe_cfg4_trace.log 2>&1
timeout 300 python tools/probe_batched.py 2 > gpurun_out/probe_cfg4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sbcg_step|k_pairs|k_rows" -s 9 -c 3 \
    -o gpurun_out/prof_cfg4_spmm python tools/probe_batched.py 2 > gpurun_out/ncu_cfg4.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_cfg3.log 2>&1
