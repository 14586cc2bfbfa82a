# ncu full captures of the finest degree-2 pass: lean vs masked
mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -o gpurun_out/r2_cheb_lean -f python tools/ncu_solve.py --config C3 --what cheb --graph 0 > gpurun_out/ncu_lean.log 2>&1
SR_FMG_CHEB_LEAN=0 timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -o gpurun_out/r2_cheb_mask -f python tools/ncu_solve.py --config C3 --what cheb --graph 0 > gpurun_out/ncu_mask.log 2>&1
