mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/gt_comb.log 2>&1; echo pytest=$? >> gpurun_out/gt_comb.log
timeout 200 python tools/probe/step_timeline.py --steps 2 > gpurun_out/tl_comb.log 2>&1
timeout 200 python tools/latency_step.py q61 9 > gpurun_out/lat_q61_comb.log 2>&1
