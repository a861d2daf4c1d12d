# N=1 headline bench, repeated (box-to-box variance is a few %)
for i in 1 2 3; do
  timeout 120 python bench.py --steps 100 --warmup 5 --no-ll --no-cpu-baseline --no-configs 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print(d['value'], d['ms_per_step'], d['kernels_ms'])
"
done
