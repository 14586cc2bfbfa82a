# ncu captures of the small-level degree-2 passes (level 6: E = 22, level 5: E = 14), fp64
mkdir -p gpurun_out
for l in 6 5; do
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -o gpurun_out/cheb_l$l -f python tools/ncu_solve.py --config C3 --what cheb --level $l --graph 0 > gpurun_out/ncu_cheb_l$l.log 2>&1
python tools/ncu_metrics.py gpurun_out/cheb_l$l.ncu-rep > gpurun_out/cheb_l${l}_metrics.txt 2>&1
done
