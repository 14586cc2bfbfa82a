# ncu capture of the level-8 fused up pass (third k_up2 launch of a solve)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_up2 --launch-skip 2 -c 1 -o gpurun_out/up2_l8 -f python tools/ncu_solve.py --graph 0 > gpurun_out/up2_ncu.log 2>&1
python tools/ncu_metrics.py gpurun_out/up2_l8.ncu-rep > gpurun_out/up2_l8_metrics.txt 2>&1
