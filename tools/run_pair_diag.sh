for v in p0 p2 p4; do echo "== $v" >> gpurun_out/suf_ab.log; HYDRA_LIB_PATH=paper_2402_05099_b200/libhydra_var_$v.so timeout 100 python tools/suffix_shapes_ab.py >> gpurun_out/suf_ab.log 2>&1; done
