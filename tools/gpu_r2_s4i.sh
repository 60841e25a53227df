# session 4, call i: ahead mode with the streaming kernel (sizes without the overlap mode) -- tests, cfg2/cfg3 probes with and without
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_resident.py tests/test_gpu_parity.py -m gpu -x -q --timeout 200 > gpurun_out/gputests_i.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_i.log
out=gpurun_out/ahead_large.txt; : > $out
for c in cfg2 cfg3; do for a in 16 0; do echo "== $c THERMO_AHEAD=$a" >> $out; THERMO_AHEAD=$a THERMO_CG_VERBOSE=1 timeout 300 python tools/probe.py $c 20 2>&1 | grep -v "^\[thermo cg\]" | tail -4 >> $out; done; done
timeout 900 python -m pytest tests/test_gpu_fullrun.py -m gpu -x -q --timeout 400 -k "cfg2 or cfg3" >> gpurun_out/gputests_i.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_i.log
