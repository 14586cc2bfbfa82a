# ncu capture of the finest-level FMG entry pass (4th k_pset1s of a solve), fp64
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_pset1s --launch-skip 3 -c 1 -o gpurun_out/ps_l8 -f python tools/ncu_solve.py --graph 0 > gpurun_out/ps_ncu.log 2>&1
python tools/ncu_metrics.py gpurun_out/ps_l8.ncu-rep > gpurun_out/ps_l8_metrics.txt 2>&1
