# robustness sweep: fused vs step kernels over (S, J, K, dtype) at 256^3 and non-cubic grids
mkdir -p gpurun_out
timeout 1500 python tools/robust_sweep.py > gpurun_out/robust.log 2>&1; echo "rc=$?" >> gpurun_out/robust.log
