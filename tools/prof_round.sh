set -x
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r1b_pytest_gpu.log 2>&1; tail -3 gpurun_out/r1b_pytest_gpu.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1b_launches_bench_steps2.csv timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r1b_bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:prefix_tc2 -s 1 -c 1 -o gpurun_out/r1b_prefix_tc2 timeout 300 python tools/prefix_one.py 0 0 > gpurun_out/r1b_ncu_prefix.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 1 -c 1 -o gpurun_out/r1b_suffix_decode timeout 300 python tools/prof_kernels.py --what suffix > gpurun_out/r1b_ncu_suffix.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:suffix_tc -s 1 -c 1 -o gpurun_out/r1b_suffix_tc timeout 300 python tools/prof_kernels.py --what suffix --suffix-impl 2 > gpurun_out/r1b_ncu_suffix_tc.log 2>&1
ls -la gpurun_out
