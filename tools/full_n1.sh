# round-end style validation on one GPU
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/f_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/f_bench_n1.json 2> gpurun_out/f_bench_n1.err
timeout 600 python bench.py --impl reference > gpurun_out/f_ref_n1.json 2> gpurun_out/f_ref_n1.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches_n1.csv python tools/run_steps.py normal 5 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dispatch_kernel -s 2 -c 1 -o gpurun_out/f_ncu_dispatch_n1 -f python tools/run_steps.py normal 4 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:combine_kernel -s 2 -c 1 -o gpurun_out/f_ncu_combine_n1 -f python tools/run_steps.py normal 4 > /dev/null 2>&1
