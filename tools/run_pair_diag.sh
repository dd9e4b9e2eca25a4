timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "suffix or composite" > gpurun_out/pytest_n8.log 2>&1; tail -2 gpurun_out/pytest_n8.log
timeout 200 python tools/suffix_shapes_ab.py > gpurun_out/n8.log 2>&1
HYDRA_LIB_PATH=paper_2402_05099_b200/libhydra_var_n16.so timeout 200 python tools/suffix_shapes_ab.py >> gpurun_out/n8.log 2>&1
timeout 300 python tools/overlap_sustained.py 60,64 >> gpurun_out/n8.log 2>&1
HYDRA_LIB_PATH=paper_2402_05099_b200/libhydra_var_n16.so timeout 300 python tools/overlap_sustained.py 60,64 >> gpurun_out/n8.log 2>&1
