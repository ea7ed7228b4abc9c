mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/gt_z20.log 2>&1; echo pytest=$? >> gpurun_out/gt_z20.log
rm -f gpurun_out/z20_all.log
for r in 1 2; do for v in h n; do
  echo "== $v" >> gpurun_out/z20_all.log
  GSLS_LIB=$PWD/paper_2604_07644_b200/libgsls_$v.so timeout 200 python tools/probe/step_timeline.py --steps 2 2>&1 | grep -E "  gains|wall" >> gpurun_out/z20_all.log
done; done
