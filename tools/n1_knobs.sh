# N=1 step under the reduce/copy work-unit knobs
for cfg in "-1" "0" "-1" "0"; do
  EPB_COMBINE_SEG16=$cfg timeout 300 python bench.py --no-configs --no-cpu-baseline --no-ll 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('seg=$cfg', d['value'], d['ms_per_step'], d['kernels_ms'], d['eager']['ms_per_step'], d['roofline']['frac'])"
done
