# N=2 combine variants (run on a 2-GPU box)
for cfg in "1 224" "1 0" "1 448" "0 0" "1 224" "1 0"; do
  set -- $cfg
  EPB_COMBINE_WIDE=$1 EPB_COMBINE_SEG16=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --no-configs --no-cpu-baseline --no-ll 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('wide=$1 seg=$2', d['value'], d['ms_per_step'], d['kernels_ms'], d['eager']['ms_per_step'])"
done
