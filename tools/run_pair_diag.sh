for c in c4_1gpu c6_longdoc c2 c5; do timeout 300 python bench.py --config $c --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1; done
