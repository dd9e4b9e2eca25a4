timeout 200 python tools/prefix_ab.py t1,6,9 c6,c2 > gpurun_out/prefix_ab.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench.log 2>&1
timeout 200 python bench.py --config c4_1gpu --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.log 2>&1
timeout 200 python bench.py --config c6_longdoc --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/bench_c6.log 2>&1
