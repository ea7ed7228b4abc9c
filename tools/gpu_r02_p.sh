mkdir -p gpurun_out
GSLS_REPLAY_STAGED=1 GSLS_ADMM_VERBOSE=1 timeout 200 python tools/probe/step_timeline.py --steps 1 > gpurun_out/tl_staged_all.log 2>&1
GSLS_REPLAY_STAGED=1 GSLS_STAGED_GROUPS=2 GSLS_ADMM_VERBOSE=1 timeout 200 python tools/probe/step_timeline.py --steps 1 > gpurun_out/tl_staged_all2.log 2>&1
