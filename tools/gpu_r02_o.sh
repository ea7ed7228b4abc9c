mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/gputest_groups.log 2>&1; echo pytest=$? >> gpurun_out/gputest_groups.log
timeout 900 python bench.py > gpurun_out/bench_r02c.log 2>&1; echo bench=$? >> gpurun_out/bench_r02c.log
