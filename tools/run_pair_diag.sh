HYDRA_TESTING=1 timeout 120 python tools/pair_trace.py 4 > gpurun_out/pair_trace.log 2>&1
