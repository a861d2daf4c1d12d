#!/bin/bash
# N=1 step time under launch knobs (cooperative launch, shared-memory carveout).
# Usage (on a GPU box): bash tools/step_knobs.sh > gpurun_out/knobs.txt
for env in "" "EPB_COOP=0" "EPB_CARVEOUT=-1" "EPB_COOP=0 EPB_CARVEOUT=-1"; do
  for rep in 1 2; do
    line=$(env $env python bench.py --no-configs --no-ll --no-cpu-baseline --steps 50 2>/dev/null | tail -1)
    python - "$env" "$line" <<'PY'
import json, sys
d = json.loads(sys.argv[2])
print(f"{sys.argv[1] or 'default':28s} graph {d['ms_per_step']*1e3:6.1f} us  eager {d['eager']['ms_per_step']*1e3:6.1f} us  "
      f"kernels {d['kernels_ms']}")
PY
  done
done
