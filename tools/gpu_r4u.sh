# packed fp32 pass v2 (aligned rhs box, shuffled x-neighbours): bitwise tests, parity, A/B, ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "packed or fp32 or full_size_c3_matches" > gpurun_out/pk2_pt.log 2>&1; echo "rc=$?" >> gpurun_out/pk2_pt.log
if grep -q "rc=0" gpurun_out/pk2_pt.log; then
bash tools/ab.sh ab/libsrfmg_base.so --dtype f32 2>&1 | grep -E "==|solve|k_cheb2 +l=8" > gpurun_out/ab_pk2.txt
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -o gpurun_out/pk2_cheb -f python tools/ncu_solve.py --config C3 --dtype f32 --what cheb --graph 0 > gpurun_out/pk2_ncu.log 2>&1
python tools/ncu_metrics.py gpurun_out/pk2_cheb.ncu-rep > gpurun_out/pk2_cheb_metrics.txt 2>&1
fi
