mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/gputest_gains.log 2>&1; echo pytest=$? >> gpurun_out/gputest_gains.log
timeout 200 python tools/probe/step_timeline.py --steps 2 > gpurun_out/tl_gains5.log 2>&1
GSLS_LIB=$PWD/paper_2604_07644_b200/libgsls_b4.so timeout 200 python tools/probe/step_timeline.py --steps 2 > gpurun_out/tl_gains4.log 2>&1
