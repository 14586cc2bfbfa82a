# C4 at the driver's scaling sizes (2, 4, 8 ranks on one GPU through the host store)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -k "c4_ranks" > gpurun_out/c4_pt.log 2>&1; echo "rc=$?" >> gpurun_out/c4_pt.log
