# A/B of testing-library variants (tools/build_variants.py) on the prefix kernel alone:
#   bash tools/run_var_ab.sh OUT "var1 var2 ..." [variants] [shapes] [reps]
out=$1; vars=$2; pv=${3:-9}; shapes=${4:-c3,c4,c6}; reps=${5:-2}
for r in $(seq $reps); do for v in $vars; do
  echo "== $v" >> $out
  HYDRA_LIB_PATH=paper_2402_05099_b200/libhydra_var_$v.so timeout 120 python tools/prefix_ab.py $pv $shapes >> $out 2>&1
done; done
