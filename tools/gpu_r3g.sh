# FMG entry pass with a producer warp (fp64 E = 70): quick solve first, then parity subset, A/B (alternating), ncu
mkdir -p gpurun_out
timeout 60 python tools/single_debug.py 512,512,512 8 64 4 2 > gpurun_out/pw_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pw_quick.log
if grep -q "done True" gpurun_out/pw_quick.log; then
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "full_size_c3 or pset or C1 or C2 or noncubic or thin or large" > gpurun_out/pw_pt.log 2>&1; echo "rc=$?" >> gpurun_out/pw_pt.log
bash tools/ab.sh ab/libsrfmg_base.so > gpurun_out/ab_pw64.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_pset1s --launch-skip 3 -c 1 -o gpurun_out/ps_l8 -f python tools/ncu_solve.py --graph 0 > gpurun_out/ps_ncu.log 2>&1
python tools/ncu_metrics.py gpurun_out/ps_l8.ncu-rep > gpurun_out/ps_l8_metrics.txt 2>&1
fi
