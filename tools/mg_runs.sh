# multi-GPU measurements (run with gpurun --gpus N): bench, LL proxy phase trace, NVLink counters
N=${1:-2}
nvidia-smi nvlink -h > gpurun_out/nvlink_help.txt 2>&1
nvidia-smi nvlink -gt d > gpurun_out/nvl_before_n$N.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus $N > gpurun_out/mg_bench_n$N.json 2> gpurun_out/mg_bench_n$N.err
nvidia-smi nvlink -gt d > gpurun_out/nvl_after_n$N.txt 2>&1
EPB_TIMEOUT_S=3 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29542 tools/trace_ll_proxy.py --calls 30 > gpurun_out/mg_trace_n$N.txt 2>&1
