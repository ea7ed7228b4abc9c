mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_lqr_admm.py -m gpu -q -k "sizes_64_to_80" > gpurun_out/gjsizes.log 2>&1
GSLS_ADMM_VERBOSE=1 GSLS_REPLAY_STAGED=0 GSLS_REPLAY_KCLUSTER=1 timeout 300 python tools/probe/step_timeline.py --steps 1 > gpurun_out/timeline_kcluster.log 2>&1
GSLS_REPLAY_STAGED=0 GSLS_REPLAY_KCLUSTER=1 timeout 300 python tools/latency_step.py q61 5 > gpurun_out/lat_kcluster.log 2>&1
timeout 300 python tools/latency_step.py q61 5 > gpurun_out/lat_staged.log 2>&1
