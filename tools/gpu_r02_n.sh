mkdir -p gpurun_out
for g in 1 2 4; do
  GSLS_STAGED_GROUPS=$g timeout 200 python tools/latency_step.py q61 9 > gpurun_out/sw_q61_$g.log 2>&1
  GSLS_STAGED_GROUPS=$g timeout 200 python tools/latency_step.py h75 9 > gpurun_out/sw_h75_$g.log 2>&1
  GSLS_STAGED_GROUPS=$g GSLS_ADMM_VERBOSE=1 timeout 200 python tools/probe/step_timeline.py --steps 1 > gpurun_out/sw_tl_$g.log 2>&1
done
GSLS_LIB=$PWD/paper_2604_07644_b200/libgsls_old.so timeout 200 python tools/latency_step.py q61 9 > gpurun_out/sw_q61_old.log 2>&1
GSLS_LIB=$PWD/paper_2604_07644_b200/libgsls_old.so timeout 200 python tools/latency_step.py h75 9 > gpurun_out/sw_h75_old.log 2>&1
