mkdir -p gpurun_out
timeout 120 tools/micro/tc_gemm > gpurun_out/tc_gemm.jsonl 2>&1; echo rc=$? >> gpurun_out/tc_gemm.jsonl
timeout 600 python tools/probe/sls_shard_at_scale.py 8 0 > gpurun_out/shard_8_0.log 2>&1
timeout 600 python tools/probe/sls_shard_at_scale.py 8 7 > gpurun_out/shard_8_7.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:k_chain -s 3 -c 6 -o gpurun_out/tc_gemm_r02 tools/micro/tc_gemm > /dev/null 2>&1
ls -la gpurun_out | tail -5
