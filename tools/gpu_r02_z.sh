mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --timeout 120 -k "sls or robust or graph or batch" > gpurun_out/gt_z.log 2>&1; echo pytest=$? >> gpurun_out/gt_z.log
for lib in libgsls_old.so libgsls.so libgsls_old.so libgsls.so; do
  GSLS_LIB=$PWD/paper_2604_07644_b200/$lib timeout 200 python tools/probe/step_timeline.py --steps 2 > gpurun_out/z_$lib.log 2>&1
  cat gpurun_out/z_$lib.log >> gpurun_out/z_all.log
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sls_gains -c 1 -o gpurun_out/slsgains_z python bench.py --steps 1 --warmup 0 --no-latency --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sls_leaf -c 1 -o gpurun_out/slsleaf_z python bench.py --steps 1 --warmup 0 --no-latency --no-cpu > /dev/null 2>&1
