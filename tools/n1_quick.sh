timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "dispatch or layout or capacity or single_rank or slot" > gpurun_out/q_tests.log 2>&1
for i in 1 2; do
  timeout 300 python bench.py --no-configs --no-cpu-baseline --no-ll 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['kernels_ms'], d['roofline']['frac'], d['eager']['ms_per_step'])"
done
