mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest3.log 2>&1; echo pytest=$? >> gpurun_out/gputest3.log
GSLS_COMBINE_TRACE=1 timeout 300 python tools/latency_step.py q61 2 1024 > gpurun_out/trace_q61b.log 2>&1
GSLS_COMBINE_TRACE=1 timeout 300 python tools/latency_step.py h75 2 256 > gpurun_out/trace_h75b.log 2>&1
timeout 300 python tools/probe/step_timeline.py --steps 2 > gpurun_out/timeline3.log 2>&1
echo done
