# Round-2 (late) profile pass (tools/profile_r2b.sh): launch list of a short C3@16K bench, ncu --set full of
# the CTA-pair prefix kernel (alone, C3@16K, pair_poly 0), the short-suffix kernel (C6 shape) and the
# tensor-core suffix on its C3 overlap share; raw pages exported as CSV next to the reports.
python -m paper_2402_05099_b200.build > /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2u_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --paged-page-size 0 > gpurun_out/r2u_launches_bench.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:prefix_pair -c 1 -o gpurun_out/r2u_pair_c3 \
  python tools/prefix_ab.py 9 c3 > gpurun_out/r2u_ncu_pair.log 2>&1
SHAPES="c6:256,32,4,128" IMPL=3 timeout 300 ncu --set full --clock-control none --import-source on -k regex:suffix_short -c 1 \
  -o gpurun_out/r2u_suffix_short_c6 python tools/suffix_shapes_ab.py > gpurun_out/r2u_ncu_short.log 2>&1
SHAPES="c4:512,32,8,128" IMPL=3 timeout 300 ncu --set full --clock-control none --import-source on -k regex:suffix_short -c 1 \
  -o gpurun_out/r2u_suffix_short_c4 python tools/suffix_shapes_ab.py > gpurun_out/r2u_ncu_short4.log 2>&1
for r in r2u_pair_c3 r2u_suffix_short_c6 r2u_suffix_short_c4; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
done
