mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/gt_final6.log 2>&1; echo pytest=$? >> gpurun_out/gt_final6.log
timeout 900 python bench.py > gpurun_out/bench_final6.log 2>&1; echo bench=$? >> gpurun_out/bench_final6.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_final6.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b1024_final6.csv python bench.py --steps 1 --warmup 1 --no-latency --no-cpu > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b1_q61_final6.csv python tools/latency_step.py q61 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sls_gains -c 1 -o gpurun_out/slsgains_final6 python bench.py --steps 1 --warmup 0 --no-latency --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sls_leaf -c 1 -o gpurun_out/slsleaf_final6 python bench.py --steps 1 --warmup 0 --no-latency --no-cpu > /dev/null 2>&1
