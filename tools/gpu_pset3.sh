mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --set full --clock-control none -k regex:k_restrict --launch-skip 6 -c 1 -o gpurun_out/r1_restrict_full -f python tools/ncu_solve.py --config C3 --what solve --graph 0 > gpurun_out/ncu_r.log 2>&1
timeout 600 ncu --profile-from-start off --set full --clock-control none -k regex:k_prolong_tma --launch-skip 9 -c 1 -o gpurun_out/r1_prolong_full -f python tools/ncu_solve.py --config C3 --what solve --graph 0 > gpurun_out/ncu_p.log 2>&1
