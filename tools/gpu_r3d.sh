# prolongation: 6 rows per thread from E = 22 on (both dtypes)
mkdir -p gpurun_out
timeout 300 python tools/breakdown.py > gpurun_out/bd_pr64.txt 2>&1
timeout 300 python tools/breakdown.py --dtype f32 > gpurun_out/bd_pr32.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "full_size_c3 or fp32 or C1 or C2 or noncubic or thin or large or c4" > gpurun_out/pr_pt.log 2>&1; echo "rc=$?" >> gpurun_out/pr_pt.log
