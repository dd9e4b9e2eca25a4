timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 400 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1
