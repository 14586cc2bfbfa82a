mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_restrict --launch-skip 3 -c 1 -o gpurun_out/restrict_full -f python tools/ncu_solve.py --config C3 --what solve --graph 0 > gpurun_out/ncu_restrict.log 2>&1
