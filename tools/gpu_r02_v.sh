mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/gt_rbase.log 2>&1; echo pytest=$? >> gpurun_out/gt_rbase.log
GSLS_REPLAY_TRACE=1 timeout 300 python tools/latency_step.py q61 2 > gpurun_out/trace_b1.log 2>&1
timeout 200 python tools/latency_step.py q61 9 > gpurun_out/lat_q61_rb.log 2>&1
timeout 200 python tools/latency_step.py h75 9 > gpurun_out/lat_h75_rb.log 2>&1
