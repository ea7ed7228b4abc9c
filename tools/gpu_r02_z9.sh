mkdir -p gpurun_out
GSLS_ADMM_LAG_MIN=2 timeout 900 python -m pytest tests -m gpu -q --timeout 120 > gpurun_out/gt_z9_lag2.log 2>&1; echo pytest=$? >> gpurun_out/gt_z9_lag2.log
rm -f gpurun_out/z9_all.log
for L in 0 296 0 296 600; do
  echo "== lag_min $L" >> gpurun_out/z9_all.log
  GSLS_ADMM_LAG_MIN=$L GSLS_OVERLAP=1 GSLS_ADMM_VERBOSE=1 timeout 200 python tools/probe/step_timeline.py --steps 1 > gpurun_out/z9_l$L.log 2>&1
  grep -E "wall" gpurun_out/z9_l$L.log >> gpurun_out/z9_all.log
  grep "admm wave" gpurun_out/z9_l$L.log | tail -50 | awk '{s+=$NF+0} END {print "waves", NR, "sum_ms", s}' >> gpurun_out/z9_all.log
  grep "admm wave [0-9]:" gpurun_out/z9_l$L.log | tail -10 >> gpurun_out/z9_all.log
done
for L in 0 296 0 296; do
  GSLS_ADMM_LAG_MIN=$L timeout 600 python bench.py --no-latency --no-cpu > gpurun_out/z9_bench_l$L.log 2>&1
  echo "lag $L $(tail -1 gpurun_out/z9_bench_l$L.log | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["e2e"]["value"])')" >> gpurun_out/z9_all.log
done
