mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r02.log 2>&1; echo pytest=$? >> gpurun_out/gputest_r02.log
timeout 900 python bench.py > gpurun_out/bench_r02.log 2>&1; echo bench=$? >> gpurun_out/bench_r02.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b1024_r02.csv python bench.py --steps 1 --warmup 1 --no-latency --no-cpu > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b1_q61_r02.csv python tools/latency_step.py q61 2 > /dev/null 2>&1
echo done
