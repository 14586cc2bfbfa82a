# A/B of E = 38 degree-2 band shapes (fp64): 19 of 3 (default), 19 of 4, 13 of 3, 10 of 4
mkdir -p gpurun_out
for rep in 1 2; do for v in 0 1 2 3; do
  echo "== e38=$v"; SR_FMG_E38=$v timeout 300 python tools/breakdown.py 2>&1 | grep -E "solve|k_cheb2 +l=7"
done; done > gpurun_out/ab_e38.txt 2>&1
SR_FMG_E38=2 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "full_size_c3_matches or C2 or c5_shapes" > gpurun_out/e38_pt.log 2>&1; echo "rc=$?" >> gpurun_out/e38_pt.log
