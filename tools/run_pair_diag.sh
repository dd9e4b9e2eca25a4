timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
CLUSTERS=1,2,4 timeout 300 python tools/pair_power.py > gpurun_out/mc_power.log 2>&1
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
