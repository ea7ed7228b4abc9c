mkdir -p gpurun_out
for g in 1 2; do
  GSLS_STAGED_GROUPS=$g timeout 200 python tools/latency_step.py q61 9 > gpurun_out/sw_q61_$g.log 2>&1
  GSLS_STAGED_GROUPS=$g timeout 200 python tools/latency_step.py h75 9 > gpurun_out/sw_h75_$g.log 2>&1
done
