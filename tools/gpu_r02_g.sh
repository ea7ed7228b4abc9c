mkdir -p gpurun_out
GSLS_TC=0 timeout 300 python tools/probe/step_timeline.py --steps 2 > gpurun_out/timeline_simt.log 2>&1
timeout 300 python tools/probe/step_timeline.py --steps 2 > gpurun_out/timeline_tc.log 2>&1
timeout 300 python tools/probe/tc_ab.py 64 > gpurun_out/tc_ab.log 2>&1
for v in 0 1; do GSLS_TC=$v timeout 600 python -m pytest tests/test_gpu_batch.py -m gpu -q > gpurun_out/tcb_$v.log 2>&1; done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_matprod -s 2 -c 1 -o gpurun_out/matprod_tc python bench.py --steps 1 --warmup 0 --no-latency --no-cpu > /dev/null 2>&1
GSLS_TC=0 timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_matprod -s 2 -c 1 -o gpurun_out/matprod_simt python bench.py --steps 1 --warmup 0 --no-latency --no-cpu > /dev/null 2>&1
