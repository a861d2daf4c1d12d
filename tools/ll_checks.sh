# LL proxy: parity tests + bench LL lines (1 GPU)
timeout 600 python -m pytest tests/test_proxy.py tests/test_gpu_parity.py tests/test_gpu_scale.py -k "ll or drain or proxy or fault" -x -q > gpurun_out/ll_tests.log 2>&1
EPB_TIMEOUT_S=3 timeout 200 python tools/trace_ll_proxy.py --calls 20 > gpurun_out/ll_trace_n1.txt 2>&1
timeout 300 python bench.py --no-configs --no-cpu-baseline > gpurun_out/ll_bench_n1.json 2> gpurun_out/ll_bench_n1.err
