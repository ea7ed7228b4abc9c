mkdir -p gpurun_out
timeout 60 tools/micro/tc_test > gpurun_out/tc_test.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_tc.log 2>&1; echo pytest=$? >> gpurun_out/gputest_tc.log
GSLS_TC=0 timeout 300 python tools/probe/step_timeline.py --steps 2 > gpurun_out/timeline_simt.log 2>&1
timeout 300 python tools/probe/step_timeline.py --steps 2 > gpurun_out/timeline_tc.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_matprod -s 2 -c 1 -o gpurun_out/matprod_tc python bench.py --steps 1 --warmup 0 --no-latency --no-cpu > /dev/null 2>&1
GSLS_TC=0 timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_matprod -s 2 -c 1 -o gpurun_out/matprod_simt python bench.py --steps 1 --warmup 0 --no-latency --no-cpu > /dev/null 2>&1
