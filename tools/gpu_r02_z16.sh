mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 120 > gpurun_out/gt_z16.log 2>&1; echo pytest=$? >> gpurun_out/gt_z16.log
rm -f gpurun_out/z16_all.log
for r in 1 2; do for v in h n; do
  echo "== $v" >> gpurun_out/z16_all.log
  GSLS_LIB=$PWD/paper_2604_07644_b200/libgsls_$v.so timeout 200 python tools/probe/step_timeline.py --steps 2 2>&1 | grep -E "sls_cvf|wall" >> gpurun_out/z16_all.log
done; done
