# SpMM sweep composition: ring depth and debug modes (THERMO_CG_TRACE=3 phase split)
mkdir -p gpurun_out
out=gpurun_out/spmm_probe.txt; : > $out
for ns in 2 3 4 5; do echo "== stages $ns" >> $out; THERMO_CGB_STAGES=$ns THERMO_CG_TRACE=3 timeout 300 python tools/probe_batched.py 3 2>&1 | tail -2 >> $out; done
for d in 1 2 8 16; do echo "== debug $d" >> $out; THERMO_CGB_DEBUG=$d THERMO_CG_TRACE=3 timeout 300 python tools/probe_batched.py 3 2>&1 | tail -2 >> $out; done
echo "== verbose" >> $out; THERMO_CG_VERBOSE=1 timeout 300 python tools/probe_batched.py 1 2>&1 | grep -i "cgb\|S=64" >> $out
