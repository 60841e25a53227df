# session 4, call c: A/B on one box -- HEAD library vs the cp.async software-pipelined sweep (2 groups x 2 stages / 1 group x 4 stages)
mkdir -p gpurun_out
out=gpurun_out/spmm_ab.txt; : > $out
run() { echo "== $1" >> $out; shift; env "$@" THERMO_CG_TRACE=3 timeout 300 python tools/probe_batched.py 5 2>&1 | tail -2 >> $out; }
timeout 900 python -m pytest tests/test_gpu_batched.py -m gpu -x -q > gpurun_out/gputests_batched.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_batched.log
run "HEAD" DIAG_LIB=tools/ab/libthermo_head.so
run "new g2"
run "new g1" DIAG_LIB=tools/ab/libthermo_g1.so
run "new g1 stages 3" DIAG_LIB=tools/ab/libthermo_g1.so THERMO_CGB_STAGES=3
run "new g1 stages 2" DIAG_LIB=tools/ab/libthermo_g1.so THERMO_CGB_STAGES=2
run "new g2 debug 1 (no row sums)" THERMO_CGB_DEBUG=1
run "new g2 debug 3 (no row sums, no windows)" THERMO_CGB_DEBUG=3
run "new g2 debug 65 (no row sums, windows only)" THERMO_CGB_DEBUG=65
run "new g2 debug 67 (no row sums, no copies)" THERMO_CGB_DEBUG=67
run "new g2 debug 103 (no row sums, no copies, no epilogue, no stores)" THERMO_CGB_DEBUG=103
run "new g1 debug 1 (no row sums)" DIAG_LIB=tools/ab/libthermo_g1.so THERMO_CGB_DEBUG=1
