timeout 900 python -m pytest tests/test_multigpu.py -q > gpurun_out/n4f_tests.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 4 > gpurun_out/n4f_bench.json 2> gpurun_out/n4f_bench.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29572 bench.py --gpus 4 --impl reference > gpurun_out/n4f_ref.json 2> gpurun_out/n4f_ref.err
EPB_TIMEOUT_S=3 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29573 tools/trace_ll_proxy.py --calls 30 > gpurun_out/n4f_trace.txt 2>&1
