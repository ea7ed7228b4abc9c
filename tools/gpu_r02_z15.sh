mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 120 > gpurun_out/gt_z15.log 2>&1; echo pytest=$? >> gpurun_out/gt_z15.log
rm -f gpurun_out/z15_all.log
for r in 1 2; do for v in h n; do
  echo "== $v" >> gpurun_out/z15_all.log
  GSLS_LIB=$PWD/paper_2604_07644_b200/libgsls_$v.so timeout 200 python tools/probe/step_timeline.py --steps 2 2>&1 | grep -E "sls_leaf|wall" >> gpurun_out/z15_all.log
done; done
for v in h n; do GSLS_LIB=$PWD/paper_2604_07644_b200/libgsls_$v.so timeout 200 python tools/latency_step.py h75 20 2>&1 | tail -1 >> gpurun_out/z15_all.log; done
