for r in 1 2; do for v in new legacy; do
  echo "== $v" >> gpurun_out/r3v_ab.log
  HYDRA_LIB_PATH=paper_2402_05099_b200/libhydra_var_$v.so KEY=seq_pdl VALUES=1 FLUSH=1 timeout 200 python tools/config_ab.py c6 >> gpurun_out/r3v_ab.log 2>&1
  HYDRA_LIB_PATH=paper_2402_05099_b200/libhydra_var_$v.so KEY=seq_pdl VALUES=1 timeout 200 python tools/config_ab.py c4 >> gpurun_out/r3v_ab.log 2>&1
done; done
