set -x
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b1024_r01f.csv python bench.py --steps 1 --warmup 1 --no-latency --no-cpu > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b1_q61_r01f.csv python tools/latency_step.py q61 2 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_cvf_combine -s 9 -c 1 -o gpurun_out/comb_r01f python bench.py --steps 1 --warmup 1 --no-latency --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_replay -c 1 -o gpurun_out/replay_r01f python bench.py --steps 1 --warmup 0 --no-latency --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_admm_staged -s 2 -c 1 -o gpurun_out/staged_r01f python tools/latency_step.py q61 3 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_rollout -c 1 -o gpurun_out/rollout_r01f python bench.py --steps 1 --warmup 0 --no-latency --no-cpu > /dev/null 2>&1
ls -la gpurun_out
