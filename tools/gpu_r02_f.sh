mkdir -p gpurun_out
for v in c m; do
  GSLS_TC=$v timeout 600 python -m pytest tests/test_gpu_batch.py -m gpu -q -x -k "q61" > gpurun_out/tcb_$v.log 2>&1
done
GSLS_OVERLAP=0 GSLS_TC=1 timeout 600 python -m pytest tests/test_gpu_batch.py -m gpu -q -x -k "q61" > gpurun_out/tcb_serial.log 2>&1
