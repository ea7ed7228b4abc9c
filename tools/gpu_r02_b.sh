mkdir -p gpurun_out
GSLS_ADMM_VERBOSE=1 timeout 300 python tools/probe/step_timeline.py --steps 2 > gpurun_out/timeline_r02.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_replay -c 1 -o gpurun_out/replay_r02 python bench.py --steps 1 --warmup 0 --no-latency --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_admm_staged -s 20 -c 1 -o gpurun_out/staged_tail_r02 python bench.py --steps 1 --warmup 0 --no-latency --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_cvf_combine -s 9 -c 1 -o gpurun_out/comb_r02 python bench.py --steps 1 --warmup 1 --no-latency --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sls_gains -c 1 -o gpurun_out/slsgains_r02 python bench.py --steps 1 --warmup 0 --no-latency --no-cpu > /dev/null 2>&1
ls -la gpurun_out
