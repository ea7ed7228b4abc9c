mkdir -p gpurun_out
rm -f gpurun_out/z21_all.log
for r in 1 2; do for v in h n5 n4; do
  echo "== $v" >> gpurun_out/z21_all.log
  GSLS_LIB=$PWD/paper_2604_07644_b200/libgsls_$v.so timeout 200 python tools/probe/step_timeline.py --steps 2 2>&1 | grep -E "sls_rownorm|wall" >> gpurun_out/z21_all.log
done; done
