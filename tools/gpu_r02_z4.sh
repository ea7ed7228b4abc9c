mkdir -p gpurun_out
rm -f gpurun_out/z4_all.log
for P in 0 1 0 1; do
  echo "== prio $P" >> gpurun_out/z4_all.log
  GSLS_SIDE_PRIORITY=$P GSLS_OVERLAP=1 GSLS_ADMM_VERBOSE=1 timeout 200 python tools/probe/step_timeline.py --steps 1 > gpurun_out/z4_p$P.log 2>&1
  grep -E "wall" gpurun_out/z4_p$P.log >> gpurun_out/z4_all.log
  grep "admm wave [0-7]:" gpurun_out/z4_p$P.log | tail -8 >> gpurun_out/z4_all.log
done
for P in 0 1; do
  GSLS_SIDE_PRIORITY=$P timeout 600 python bench.py --no-latency --no-cpu > gpurun_out/z4_bench_p$P.log 2>&1
done
