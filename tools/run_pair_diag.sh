timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "scatter or p2p or seqsplit or combine" > gpurun_out/pytest_p2p.log 2>&1; tail -15 gpurun_out/pytest_p2p.log
