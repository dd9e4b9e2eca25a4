for k in 56 60 64 68; do timeout 300 python bench.py --no-cpu-baseline --no-e2e --paged-page-size 0 --overlap-k $k > gpurun_out/bench_k$k.log 2>&1; done
