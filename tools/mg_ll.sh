N=${1:-2}
for sig in writevalue memcpy writevalue memcpy; do
EPB_PROXY_SIGNAL=$sig EPB_TIMEOUT_S=3 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29545 tools/trace_ll_proxy.py --calls 20 --fifo-channels 16 2>/dev/null | grep "^{" | sed "s/^{/{\"sig\": \"$sig\", /" >> gpurun_out/mgll_trace_n$N.txt
done
