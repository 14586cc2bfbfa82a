# deeper u0 / rhs rings for the E = 22 / 14 degree-2 passes: quick solve, parity subset, A/B (alternating) fp64 and fp32
mkdir -p gpurun_out
timeout 60 python tools/single_debug.py 512,512,512 8 64 4 2 > gpurun_out/rr_quick.log 2>&1; echo "rc=$?" >> gpurun_out/rr_quick.log
if grep -q "done True" gpurun_out/rr_quick.log; then
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "full_size_c3 or pset or C1 or C2 or noncubic or thin or tau or fp32" > gpurun_out/rr_pt.log 2>&1; echo "rc=$?" >> gpurun_out/rr_pt.log
bash tools/ab.sh ab/libsrfmg_base.so > gpurun_out/ab_rr64.txt 2>&1
bash tools/ab.sh ab/libsrfmg_base.so --dtype f32 > gpurun_out/ab_rr32.txt 2>&1
fi
