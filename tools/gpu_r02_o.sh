mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/gputest_groups.log 2>&1; echo pytest=$? >> gpurun_out/gputest_groups.log
timeout 900 python bench.py > gpurun_out/bench_r02d.log 2>&1; echo bench=$? >> gpurun_out/bench_r02d.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_admm_staged -s 1 -c 1 -o gpurun_out/staged_bulk_r02 python bench.py --steps 1 --warmup 0 --no-latency --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b1024_r02d.csv python bench.py --steps 1 --warmup 1 --no-latency --no-cpu > /dev/null 2>&1
