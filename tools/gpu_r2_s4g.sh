# session 4, call g: resident sweep with two volume rows per thread group in flight -- cfg1 forced, small sizes, tests
mkdir -p gpurun_out
out=gpurun_out/resident_cfg1.txt; : > $out
THERMO_CG_RESIDENT=1 THERMO_CG_TRACE=1 timeout 120 python tools/probe.py cfg1 20 2>&1 | grep -v "^\[thermo c" | tail -4 >> $out
THERMO_CG_TRACE=1 timeout 120 python tools/probe.py cfg1 20 2>&1 | grep -v "^\[thermo c" | tail -4 >> $out
for c in cfg0 medium; do THERMO_CG_TRACE=1 timeout 120 python tools/probe.py $c 20 2>&1 | grep -v "^\[thermo c" | tail -4; done >> $out
timeout 500 python -m pytest tests/test_gpu_resident.py -m gpu -x -q --timeout 150 > gpurun_out/gputests_g.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_g.log
