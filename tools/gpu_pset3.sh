mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_up2s --launch-skip 2 -c 1 -o gpurun_out/up_full -f python tools/ncu_solve.py --config C3 --what solve --graph 0 > gpurun_out/ncu_up.log 2>&1
