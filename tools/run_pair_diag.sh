timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
KEY=seq_pdl VALUES=0,1 timeout 300 python tools/config_ab.py > gpurun_out/seq_pdl.log 2>&1
for c in c4_1gpu c6_longdoc c2; do timeout 300 python bench.py --config $c --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1; done
