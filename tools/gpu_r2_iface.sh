# interface single-sided pairs: full GPU suite + probes
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/gputests.log 2>&1; echo "rc=$?" >> gpurun_out/gputests.log
timeout 300 python tools/probe_batched.py 5 > gpurun_out/probe_cfg4.log 2>&1
out=gpurun_out/spmm_probe2.txt; : > $out
for d in 3 9 11; do echo "== debug $d" >> $out; THERMO_CGB_DEBUG=$d THERMO_CG_TRACE=3 timeout 300 python tools/probe_batched.py 3 2>&1 | tail -2 >> $out; done
