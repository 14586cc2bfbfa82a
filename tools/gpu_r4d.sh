# packed fp32 degree-2 pass (k_cheb2p): bitwise vs the scalar lean pass, fp32 parity, A/B timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "packed or fp32 or full_size_c3_matches or fused_and_step" > gpurun_out/pk_pt.log 2>&1; echo "rc=$?" >> gpurun_out/pk_pt.log
for rep in 1 2; do
  echo "== scalar $rep"; SR_FMG_CHEB_PACK=0 timeout 300 python tools/breakdown.py --dtype f32 | head -9
  echo "== packed $rep"; SR_FMG_CHEB_PACK=1 timeout 300 python tools/breakdown.py --dtype f32 | head -9
done > gpurun_out/ab_pack.txt 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -o gpurun_out/pk_cheb -f python tools/ncu_solve.py --config C3 --dtype f32 --what cheb --graph 0 > gpurun_out/pk_ncu.log 2>&1
python tools/ncu_metrics.py gpurun_out/pk_cheb.ncu-rep > gpurun_out/pk_cheb_metrics.txt 2>&1
