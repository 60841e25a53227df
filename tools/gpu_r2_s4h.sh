# session 4, call h: full GPU suite at the resident/ahead commit, smoke, ncu of the resident kernel (medium), bench lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 --durations=8 > gpurun_out/gputests.log 2>&1; echo "rc=$?" >> gpurun_out/gputests.log
timeout 200 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 200 python tools/probe.py medium 20 > gpurun_out/probe_medium.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_cg_resident|k_pairs|k_rows|k_refsort" -s 20 -c 6 \
    -o gpurun_out/prof_resident_medium python tools/probe.py medium 20 > gpurun_out/ncu_resident.log 2>&1
timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 > gpurun_out/bench_cfg4.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_cfg3.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg3.log
