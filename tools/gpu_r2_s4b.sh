# session 4, call b: lane-per-row SpMM consumers -- batched tests, probe, phase trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batched.py -m gpu -x -q > gpurun_out/gputests_batched.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_batched.log
timeout 300 python tools/probe_batched.py 5 > gpurun_out/probe_cfg4.log 2>&1
THERMO_CG_TRACE=3 timeout 300 python tools/probe_batched.py 5 > gpurun_out/probe_cfg4_trace.log 2>&1
out=gpurun_out/spmm_debug_modes.txt; : > $out
for d in 1 2 4 8 32 33; do echo "== debug $d" >> $out; THERMO_CGB_DEBUG=$d THERMO_CG_TRACE=3 timeout 300 python tools/probe_batched.py 3 2>&1 | tail -2 >> $out; done
