mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/gt_bphys.log 2>&1; echo pytest=$? >> gpurun_out/gt_bphys.log
GSLS_REPLAY_VERBOSE=1 timeout 300 python tools/latency_step.py q61 1 1024 > gpurun_out/v_b1024.log 2>&1
GSLS_ADMM_VERBOSE=1 timeout 200 python tools/probe/step_timeline.py --steps 1 > gpurun_out/tl_bphys.log 2>&1
timeout 200 python tools/latency_step.py q61 9 > gpurun_out/lat_q61_bphys.log 2>&1
timeout 200 python tools/latency_step.py h75 9 > gpurun_out/lat_h75_bphys.log 2>&1
