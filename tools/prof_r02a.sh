mkdir -p gpurun_out
GSLS_PLAN_VERBOSE=1 GSLS_COMBINE_TRACE=1 timeout 300 python tools/latency_step.py q61 2 1024 > gpurun_out/trace_q61.log 2>&1
GSLS_PLAN_VERBOSE=1 GSLS_COMBINE_TRACE=1 timeout 300 python tools/latency_step.py h75 2 256 > gpurun_out/trace_h75.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_cvf_combine -s 9 -c 1 -o gpurun_out/comb_fact_r02 python bench.py --steps 1 --warmup 1 --no-latency --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_cvf_combine -s 17 -c 1 -o gpurun_out/comb_last_r02 python bench.py --steps 1 --warmup 1 --no-latency --no-cpu > /dev/null 2>&1
echo done
