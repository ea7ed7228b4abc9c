mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 120 > gpurun_out/gt_z3.log 2>&1; echo pytest=$? >> gpurun_out/gt_z3.log
rm -f gpurun_out/z3_all.log
for r in 1 2; do for v in base v1 v4; do
  echo "== $v" >> gpurun_out/z3_all.log
  GSLS_LIB=$PWD/paper_2604_07644_b200/libgsls_$v.so timeout 200 python tools/probe/step_timeline.py --steps 2 2>&1 | grep -E "sls_leaf|sls_gains|wall|  leaf|  gains|cvf_lqr" >> gpurun_out/z3_all.log
  GSLS_LIB=$PWD/paper_2604_07644_b200/libgsls_$v.so timeout 200 python tools/latency_step.py q61 30 2>&1 | tail -2 >> gpurun_out/z3_all.log
done; done
