EPB_TMA=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q -k "dispatch_combine or dsv3_normal or qwen3 or single_rank or fp8_tuple" > gpurun_out/tc_tests_tma.log 2>&1
for i in 1; do timeout 300 python bench.py --no-cpu-baseline --no-ll 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['kernels_ms'], d['roofline']['frac'], d['sm_budget'], d['verified']['verified'])"; done > gpurun_out/tc_bench.txt 2>&1
