mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/gputest_groups.log 2>&1; echo pytest=$? >> gpurun_out/gputest_groups.log
GSLS_ADMM_VERBOSE=1 timeout 200 python tools/probe/step_timeline.py --steps 1 > gpurun_out/timeline_groups.log 2>&1
GSLS_REPLAY_VERBOSE=1 timeout 200 python tools/latency_step.py q61 7 > gpurun_out/lat_groups.log 2>&1
GSLS_REPLAY_VERBOSE=1 GSLS_ADMM_VERBOSE=1 timeout 200 python tools/probe/step_timeline.py --steps 1 --batch 64 > gpurun_out/timeline_b64.log 2>&1
