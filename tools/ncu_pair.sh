# one ncu --set full capture of the CTA-pair prefix kernel at C3@16K (tools/prefix_ab.py)
timeout 300 ncu --set full --clock-control none --import-source on -k regex:prefix_pair -c 1 -o gpurun_out/r2_pair_c3 python tools/prefix_ab.py 9 c3 > gpurun_out/ncu_pair.log 2>&1
