# rhs kept in registers between the two stages of the degree-2 passes: parity, A/B fp64 + fp32
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "full_size_c3_matches or packed or fused_and_step or tau or C2 or solve_matches or fp32 or kernel_cheb" > gpurun_out/freg_pt.log 2>&1; echo "rc=$?" >> gpurun_out/freg_pt.log
if grep -q "rc=0" gpurun_out/freg_pt.log; then
bash tools/ab.sh ab/libsrfmg_base.so 2>&1 | grep -E "==|solve|k_cheb2 +l=[5678]" > gpurun_out/ab_freg64.txt
bash tools/ab.sh ab/libsrfmg_base.so --dtype f32 2>&1 | grep -E "==|solve|k_cheb2 +l=[5678]" > gpurun_out/ab_freg32.txt
fi
