# Late round-2 pass 2 (tools/profile_r3.sh): ncu --set full of the CTA-pair prefix kernel at the C4 and C6
# shapes (the dominant kernel of those steps), raw pages exported as CSV.
python -m paper_2402_05099_b200.build > /dev/null
for s in c4 c6; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:prefix_pair -c 1 -o gpurun_out/r3_pair_$s \
    python tools/prefix_ab.py 9 $s > gpurun_out/r3_ncu_pair_$s.log 2>&1
  ncu -i gpurun_out/r3_pair_$s.ncu-rep --page raw --csv > gpurun_out/r3_pair_${s}_raw.csv 2>/dev/null
done
