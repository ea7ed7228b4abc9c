mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_rti.log 2>&1; echo pytest=$? >> gpurun_out/gputest_rti.log
timeout 300 python tools/probe/step_timeline.py --steps 2 > gpurun_out/timeline_rti.log 2>&1
timeout 300 python tools/latency_step.py q61 5 > gpurun_out/lat_rti.log 2>&1
