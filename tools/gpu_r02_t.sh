mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r02e.log 2>&1; echo bench=$? >> gpurun_out/bench_r02e.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_admm_staged -c 1 -o gpurun_out/staged_bulk_r02e python bench.py --steps 1 --warmup 0 --no-latency --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b1024_r02e.csv python bench.py --steps 1 --warmup 1 --no-latency --no-cpu > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b1_q61_r02e.csv python tools/latency_step.py q61 2 > /dev/null 2>&1
