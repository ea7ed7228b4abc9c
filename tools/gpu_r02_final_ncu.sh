mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_cvf_combine -s 9 -c 1 -o gpurun_out/comb_final python bench.py --steps 1 --warmup 1 --no-latency --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sls_gains -c 1 -o gpurun_out/slsgains_final python bench.py --steps 1 --warmup 0 --no-latency --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sls_leaf -c 1 -o gpurun_out/slsleaf_final python bench.py --steps 1 --warmup 0 --no-latency --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_admm_staged -s 3 -c 1 -o gpurun_out/staged_b1_final python tools/latency_step.py q61 3 > /dev/null 2>&1
