mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r02b.log 2>&1; echo bench=$? >> gpurun_out/bench_r02b.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_r02.log 2>&1; echo ref=$? >> gpurun_out/bench_ref_r02.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b1024_r02b.csv python bench.py --steps 1 --warmup 1 --no-latency --no-cpu > /dev/null 2>&1
