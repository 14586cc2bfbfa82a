# fused up pass: parity subset, then A/B breakdowns and an ncu capture of the level-8 pass
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "up_pass or full_size_c3 or fp32" > gpurun_out/up_pt.log 2>&1; echo "rc=$?" >> gpurun_out/up_pt.log
timeout 300 python tools/breakdown.py > gpurun_out/bd_up64.txt 2>&1
timeout 300 python tools/breakdown.py --dtype f32 > gpurun_out/bd_up32.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_up2 --launch-skip 2 -c 1 -o gpurun_out/up2_l8 -f python tools/ncu_solve.py --graph 0 > gpurun_out/up2_ncu.log 2>&1
python tools/ncu_metrics.py gpurun_out/up2_l8.ncu-rep > gpurun_out/up2_l8_metrics.txt 2>&1
