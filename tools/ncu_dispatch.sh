# ncu captures of the N=1 step kernels (one GPU): launch list + full sets of dispatch and combine
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_n1.csv python tools/run_steps.py normal 5 > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dispatch_kernel -s 2 -c 1 -o gpurun_out/ncu_dispatch_n1 -f python tools/run_steps.py normal 4 > gpurun_out/ncu_d.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:combine_kernel -s 2 -c 1 -o gpurun_out/ncu_combine_n1 -f python tools/run_steps.py normal 4 > gpurun_out/ncu_c.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:layout -s 2 -c 1 -o gpurun_out/ncu_layout_n1 -f python tools/run_steps.py normal 4 > gpurun_out/ncu_l.log 2>&1
