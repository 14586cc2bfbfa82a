# degree-2 pass with a producer warp (fp64 E = 70): quick solve, parity subset, A/B (alternating) vs the pset-PW build, ncu
mkdir -p gpurun_out
timeout 60 python tools/single_debug.py 512,512,512 8 64 4 2 > gpurun_out/cpw_quick.log 2>&1; echo "rc=$?" >> gpurun_out/cpw_quick.log
if grep -q "done True" gpurun_out/cpw_quick.log; then
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "full_size_c3 or pset or C1 or C2 or noncubic or thin or large or tau" > gpurun_out/cpw_pt.log 2>&1; echo "rc=$?" >> gpurun_out/cpw_pt.log
bash tools/ab.sh ab/libsrfmg_pw.so > gpurun_out/ab_cpw64.txt 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -o gpurun_out/cpw_cheb -f python tools/ncu_solve.py --config C3 --what cheb --graph 0 > gpurun_out/cpw_ncu.log 2>&1
python tools/ncu_metrics.py gpurun_out/cpw_cheb.ncu-rep > gpurun_out/cpw_cheb_metrics.txt 2>&1
fi
