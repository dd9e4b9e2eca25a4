timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "pair or growing or composite or fused or partitioned" > gpurun_out/pytest_pdl.log 2>&1; tail -2 gpurun_out/pytest_pdl.log
timeout 400 python bench.py --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1
timeout 300 python tools/overlap_sustained.py 52,56,60,64,68,72 > gpurun_out/ov_sus.log 2>&1
