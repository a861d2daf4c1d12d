set -x
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --no-configs --no-cpu-baseline > gpurun_out/n2_bench.json 2> gpurun_out/n2_bench.err
EPB_TIMEOUT_S=3 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 tools/trace_ll_proxy.py --calls 20 > gpurun_out/n2_trace.txt 2>&1
EPB_LL_GROUPS_PER_RANK=4 EPB_TIMEOUT_S=3 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 tools/trace_ll_proxy.py --calls 20 --fifo-channels 32 >> gpurun_out/n2_trace.txt 2>&1
timeout 600 python -m pytest tests/test_multigpu.py tests/test_proxy.py -x -q > gpurun_out/n2_tests.log 2>&1
