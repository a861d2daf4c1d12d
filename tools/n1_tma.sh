for v in 2 1 0 2 1 0; do
  EPB_TMA=$v timeout 300 python bench.py --no-cpu-baseline --no-ll 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('tma=$v', d['value'], d['ms_per_step'], d['kernels_ms'], d['roofline']['frac'], {k:(v['dispatch_us']) for k,v in d['sm_budget'].items()}, d['verified']['verified'], d['configs']['dsv3_fp8_dispatch']['dispatch_us'], d['configs']['qwen3_235b_zipf']['dispatch_us'], d['eager']['ms_per_step'])"
done
