mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_pset1s --launch-skip 1 -c 1 -o gpurun_out/pset8_full -f python tools/ncu_solve.py --config C3 --what solve --graph 0 > gpurun_out/ncu_pset.log 2>&1
