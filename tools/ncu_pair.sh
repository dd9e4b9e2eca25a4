python -c "
import paper_2402_05099_b200 as h; print('pair_max_ctas', h.get_config('pair_max_ctas'))" > gpurun_out/pair_info.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:prefix_pair -c 1 -o gpurun_out/r2_pair_c3 python tools/prefix_ab.py 9 c3 > gpurun_out/ncu_pair.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:prefix_tc2 -c 1 -o gpurun_out/r2_tc2_c3 python tools/prefix_ab.py 6 c3 >> gpurun_out/ncu_pair.log 2>&1
