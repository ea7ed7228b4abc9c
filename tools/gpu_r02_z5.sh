mkdir -p gpurun_out
for k in k_leaf_init k_gains k_sls_assemble k_sls_rownorm k_matprod; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^(gsls::)?$k\b" -c 1 -o gpurun_out/z5_$k python bench.py --steps 1 --warmup 0 --no-latency --no-cpu > gpurun_out/z5_$k.log 2>&1
done
