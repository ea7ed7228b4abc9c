mkdir -p gpurun_out
for g in 1 2 4; do GSLS_STAGED_GROUPS=$g GSLS_ADMM_VERBOSE=1 timeout 200 python tools/probe/step_timeline.py --steps 1 > gpurun_out/tlg_$g.log 2>&1; done
