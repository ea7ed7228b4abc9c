mkdir -p gpurun_out
for lib in libgsls.so libgsls_lb4.so libgsls_lb5.so; do
  GSLS_LIB=$PWD/paper_2604_07644_b200/$lib timeout 200 python tools/probe/step_timeline.py --steps 2 > gpurun_out/lb_$lib.log 2>&1
done
