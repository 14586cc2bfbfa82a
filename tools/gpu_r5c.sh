# ncu full capture of the finest 27-point degree-2 pass (P27) after the shared row sums
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -o gpurun_out/p27_cheb -f python tools/ncu_solve.py --config P27 --stencil 27pt --what cheb --graph 0 > gpurun_out/p27_ncu.log 2>&1
python tools/ncu_metrics.py gpurun_out/p27_cheb.ncu-rep > gpurun_out/p27_cheb_metrics.txt 2>&1
