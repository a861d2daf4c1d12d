N=${1:-2}
for gpd in 1 2; do
EPB_LL_GROUPS_PER_RANK=$gpd EPB_TIMEOUT_S=3 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$gpd tools/trace_ll_proxy.py --calls 20 --fifo-channels 16 2>&1 | grep "^{" >> gpurun_out/mgll_trace_n$N.txt
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29549 bench.py --gpus $N > gpurun_out/mg_bench_n$N.json 2> gpurun_out/mg_bench_n$N.err
