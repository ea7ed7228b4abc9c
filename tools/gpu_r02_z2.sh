mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --timeout 120 -k "sls or robust or graph or batch" > gpurun_out/gt_z2.log 2>&1; echo pytest=$? >> gpurun_out/gt_z2.log
rm -f gpurun_out/z2_all.log
for r in 1 2; do for v in base v1 v2 v3; do
  echo "== $v" >> gpurun_out/z2_all.log
  GSLS_LIB=$PWD/paper_2604_07644_b200/libgsls_$v.so timeout 200 python tools/probe/step_timeline.py --steps 2 2>&1 | grep -E "sls_leaf|sls_gains|wall" >> gpurun_out/z2_all.log
done; done
