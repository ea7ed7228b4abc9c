mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/gt_comb.log 2>&1; echo pytest=$? >> gpurun_out/gt_comb.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_gains.csv python bench.py --steps 1 --warmup 0 --no-latency --no-cpu > /dev/null 2>&1
