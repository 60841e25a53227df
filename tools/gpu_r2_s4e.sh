# session 4, call e: resident-operator latency solve + ahead mode -- latency probe, then the parity suites (short timeouts: a hang must not eat the budget)
mkdir -p gpurun_out
THERMO_CG_VERBOSE=1 timeout 300 python tools/probe_latency.py 50 > gpurun_out/latency_small_configs.txt 2>&1; echo "rc=$?" >> gpurun_out/latency_small_configs.txt
for c in cfg0 cfg1; do THERMO_CG_TRACE=1 timeout 120 python tools/probe.py $c 20 2>&1 | grep -v "^\[thermo c" | tail -4; done > gpurun_out/probe_resident_trace.txt
THERMO_AHEAD=0 timeout 120 python tools/probe.py cfg1 20 2>&1 | grep -v "^\[thermo c" | tail -3 >> gpurun_out/probe_resident_trace.txt
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -x -q --timeout 120 > gpurun_out/gputests_e.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_e.log
timeout 400 python -m pytest tests/test_gpu_stationary.py tests/test_gpu_mrsdc.py tests/test_gpu_sdc.py tests/test_c_abi.py tests/test_gpu_reorder.py -m gpu -x -q --timeout 120 >> gpurun_out/gputests_e.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_e.log
timeout 500 python -m pytest tests/test_gpu_fullrun.py -m gpu -x -q --timeout 200 -k "cfg1" >> gpurun_out/gputests_e.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_e.log
