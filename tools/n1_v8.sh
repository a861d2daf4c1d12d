for v in 1 0 1 0; do
  EPB_V8=$v timeout 300 python bench.py --no-configs --no-cpu-baseline --no-ll 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('v8=$v', d['value'], d['ms_per_step'], d['kernels_ms'], d['roofline']['frac'])"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dispatch_kernel -s 2 -c 1 -o gpurun_out/ncu_dispatch_v8 -f python tools/run_steps.py normal 4 > gpurun_out/ncu_d8.log 2>&1
