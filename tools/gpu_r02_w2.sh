mkdir -p gpurun_out
GSLS_OVERLAP=1 GSLS_ADMM_VERBOSE=1 timeout 300 python tools/probe/step_timeline.py --steps 1 > gpurun_out/waves_overlap.log 2>&1
