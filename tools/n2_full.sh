timeout 900 python -m pytest tests -m gpu -q > gpurun_out/n2f_tests.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 > gpurun_out/n2f_bench.json 2> gpurun_out/n2f_bench.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 2 --impl reference > gpurun_out/n2f_ref.json 2> gpurun_out/n2f_ref.err
