# ncu capture of the finest-level bulk-copy restriction (7th k_restrict_s launch of a solve), fp64 and fp32
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_restrict_s --launch-skip 6 -c 1 -o gpurun_out/rs_l8 -f python tools/ncu_solve.py --graph 0 > gpurun_out/rs_ncu.log 2>&1
python tools/ncu_metrics.py gpurun_out/rs_l8.ncu-rep > gpurun_out/rs_l8_metrics.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_restrict_s --launch-skip 6 -c 1 -o gpurun_out/rs_l8_32 -f python tools/ncu_solve.py --graph 0 --dtype f32 > gpurun_out/rs_ncu32.log 2>&1
python tools/ncu_metrics.py gpurun_out/rs_l8_32.ncu-rep > gpurun_out/rs_l8_32_metrics.txt 2>&1
