# ncu evidence for a round: R=<tag> bash tools/prof_round.sh  (run under gpurun; writes gpurun_out/)
R=${R:-r1e}
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches_bench_steps2.csv timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${R}_bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:prefix_tc2 -s 1 -c 1 -o gpurun_out/${R}_prefix_tc2 timeout 300 python tools/prefix_one.py 4 0 > gpurun_out/${R}_ncu_prefix.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:suffix_tc -s 1 -c 1 -o gpurun_out/${R}_suffix_tc_76 timeout 300 python tools/prof_kernels.py --what suffix --suffix-impl 2 --suffix-ctas 76 > gpurun_out/${R}_ncu_suffix_tc.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 1 -c 1 -o gpurun_out/${R}_suffix_decode timeout 300 python tools/prof_kernels.py --what suffix > gpurun_out/${R}_ncu_suffix.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:suffix_tc -s 1 -c 1 -o gpurun_out/${R}_suffix_tc_76_paged16 timeout 300 python tools/prof_kernels.py --what suffix --suffix-impl 2 --suffix-ctas 76 --paged 16 > gpurun_out/${R}_ncu_suffix_tc_paged.log 2>&1
ls -la gpurun_out
