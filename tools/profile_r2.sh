# Round-2 profile pass (tools/profile_r2.sh): launch list of a short bench, ncu --set full of the
# CTA-pair prefix kernel (alone, C3@16K) and of the tensor-core suffix on its overlap SM share.
python -m paper_2402_05099_b200.build > /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --paged-page-size 0 > gpurun_out/r2_launches_bench.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:prefix_pair -c 1 -o gpurun_out/r2_pair_c3 \
  python tools/prefix_ab.py 9 c3 > gpurun_out/r2_ncu_pair.log 2>&1
SUFFIX_CTAS=84 timeout 300 ncu --set full --clock-control none --import-source on -k regex:suffix_tc -c 1 -o gpurun_out/r2_suffix_tc_84 \
  python tools/suffix_alone.py > gpurun_out/r2_ncu_suffix.log 2>&1
