export SR_FMG_FORCE_FUSED=0
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pass --launch-skip 3 --launch-count 5 -o gpurun_out/pass_full -f python tools/dbg_pass.py 1 4 512 > gpurun_out/ncu_pass.log 2>&1
echo rc=$? >> gpurun_out/ncu_pass.log
