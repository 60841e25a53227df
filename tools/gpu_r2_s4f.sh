# session 4, call f: resident solve + ahead mode -- new tests, affected suites, latency probe
mkdir -p gpurun_out
timeout 500 python -m pytest tests/test_gpu_resident.py -m gpu -x -q --timeout 150 > gpurun_out/gputests_f.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_f.log
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_c_abi.py -m gpu -x -q --timeout 120 >> gpurun_out/gputests_f.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_f.log
THERMO_CG_VERBOSE=1 timeout 300 python tools/probe_latency.py 50 2>&1 | grep -v "^\[thermo cg\] \(window\|variant\|cluster\)" > gpurun_out/latency_small_configs.txt; echo "rc=$?" >> gpurun_out/latency_small_configs.txt
for c in cfg0 medium; do THERMO_CG_TRACE=1 timeout 120 python tools/probe.py $c 20 2>&1 | grep -v "^\[thermo c" | tail -4; done > gpurun_out/probe_resident_trace.txt
