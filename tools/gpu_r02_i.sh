mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_deadb.log 2>&1; echo pytest=$? >> gpurun_out/gputest_deadb.log
timeout 300 python tools/probe/step_timeline.py --steps 2 > gpurun_out/timeline_deadb.log 2>&1
