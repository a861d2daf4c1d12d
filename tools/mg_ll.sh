# LL proxy phase trace at N GPUs (tools/trace_ll_proxy.py), twice
N=${1:-2}
for rep in 1 2; do
EPB_TIMEOUT_S=3 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29545 tools/trace_ll_proxy.py --calls 20 --fifo-channels 16 2>>gpurun_out/mgll_trace_n$N.err | grep "^{" >> gpurun_out/mgll_trace_n$N.txt
done
