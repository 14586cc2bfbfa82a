# bulk-copy-fed SR restriction: parity, breakdowns, ncu capture of the finest restriction
mkdir -p gpurun_out
SR_FMG_SYNC=1 timeout 120 python tools/single_debug.py 512,512,512 8 64 4 2 > gpurun_out/rs_sync.log 2>&1; echo "rc=$?" >> gpurun_out/rs_sync.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "restrict_seg or full_size_c3 or fp32 or C1 or C2 or noncubic or thin" > gpurun_out/rs_pt.log 2>&1; echo "rc=$?" >> gpurun_out/rs_pt.log
timeout 300 python tools/breakdown.py > gpurun_out/bd_rs64.txt 2>&1
timeout 300 python tools/breakdown.py --dtype f32 > gpurun_out/bd_rs32.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_restrict_s --launch-skip 6 -c 1 -o gpurun_out/rs_l8 -f python tools/ncu_solve.py --graph 0 > gpurun_out/rs_ncu.log 2>&1
python tools/ncu_metrics.py gpurun_out/rs_l8.ncu-rep > gpurun_out/rs_l8_metrics.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_restrict_s --launch-skip 6 -c 1 -o gpurun_out/rs_l8_32 -f python tools/ncu_solve.py --graph 0 --dtype f32 > gpurun_out/rs_ncu32.log 2>&1
python tools/ncu_metrics.py gpurun_out/rs_l8_32.ncu-rep > gpurun_out/rs_l8_32_metrics.txt 2>&1
