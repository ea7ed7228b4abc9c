mkdir -p gpurun_out
GSLS_ADMM_VERBOSE=1 GSLS_REPLAY_STAGED=0 timeout 300 python tools/probe/step_timeline.py --steps 1 > gpurun_out/timeline_nostaged.log 2>&1
