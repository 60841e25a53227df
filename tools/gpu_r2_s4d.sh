# session 4, call d: batched e2e probe (state buffer released after the gather kernel, not after the DMA)
mkdir -p gpurun_out
timeout 600 python tools/probe_e2e.py 20 > gpurun_out/probe_e2e_cfg4.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_reorder.py tests/test_gpu_batched.py -m gpu -x -q > gpurun_out/gputests_d.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_d.log
timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 > gpurun_out/bench_cfg4.log 2>&1
