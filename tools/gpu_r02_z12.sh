mkdir -p gpurun_out
GSLS_COMBINE_TRACE=1 timeout 300 python tools/probe/step_timeline.py --steps 1 > gpurun_out/z12_trace.log 2>&1
