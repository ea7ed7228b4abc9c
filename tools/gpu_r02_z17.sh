mkdir -p gpurun_out
GSLS_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 3 --warmup 3 --batch 64 --no-cpu --rh-steps 20 > gpurun_out/bench_w2_gloo.log 2>&1; echo rc=$? >> gpurun_out/bench_w2_gloo.log
