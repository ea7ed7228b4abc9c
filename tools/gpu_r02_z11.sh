mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 120 > gpurun_out/gt_z11.log 2>&1; echo pytest=$? >> gpurun_out/gt_z11.log
rm -f gpurun_out/z11_all.log
for Bv in h n h n; do
  echo "== lib $Bv" >> gpurun_out/z11_all.log
  GSLS_LIB=$PWD/paper_2604_07644_b200/libgsls_$Bv.so GSLS_OVERLAP=1 GSLS_ADMM_VERBOSE=1 timeout 200 python tools/probe/step_timeline.py --steps 1 > gpurun_out/z11_b$Bv.log 2>&1
  grep -E "wall|  leaf|  gains" gpurun_out/z11_b$Bv.log >> gpurun_out/z11_all.log
  grep "admm wave" gpurun_out/z11_b$Bv.log | tail -50 | python3 -c "import sys; t=[float(l.split(':')[-1].split()[0]) for l in sys.stdin]; print('waves', len(t), 'sum', round(sum(t),2), 'tail(7+)', round(sum(t[7:]),2))" >> gpurun_out/z11_all.log
done
for Bv in h n h n; do
  GSLS_LIB=$PWD/paper_2604_07644_b200/libgsls_$Bv.so timeout 600 python bench.py --no-latency --no-cpu > gpurun_out/z11_bench_b$Bv.log 2>&1
  echo "lib $Bv $(tail -1 gpurun_out/z11_bench_b$Bv.log | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["e2e"]["value"])')" >> gpurun_out/z11_all.log
done
