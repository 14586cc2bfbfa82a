# executor index math (power-of-two shifts): parity subset, A/B (alternating builds) fp64 + fp32
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x -k "C1 or C2 or noncubic or thin or coarse or executor or full_size_c3_matches or dd or kernel" > gpurun_out/cx_pt.log 2>&1; echo "rc=$?" >> gpurun_out/cx_pt.log
bash tools/ab.sh ab/libsrfmg_base.so 2>&1 | grep -E "==|solve|k_coarse" > gpurun_out/ab_cx64.txt
bash tools/ab.sh ab/libsrfmg_base.so --dtype f32 2>&1 | grep -E "==|solve|k_coarse" > gpurun_out/ab_cx32.txt
