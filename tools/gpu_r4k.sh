# A/B: small boxes (E = 22, 14) in two bands (SR_FMG_SMALL_SPLIT=1) vs one; parity with the split
mkdir -p gpurun_out
SR_FMG_SMALL_SPLIT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "full_size_c3_matches or C2 or c5_shapes or fused_and_step or solve_matches" > gpurun_out/split_pt.log 2>&1; echo "rc=$?" >> gpurun_out/split_pt.log
for rep in 1 2; do
  for v in 0 1; do
    echo "== split=$v rep $rep f64"; SR_FMG_SMALL_SPLIT=$v timeout 300 python tools/breakdown.py 2>&1 | grep -E "solve|l=[56]"
  done
done > gpurun_out/ab_split.txt 2>&1
for v in 0 1; do
  echo "== split=$v f32"; SR_FMG_SMALL_SPLIT=$v timeout 300 python tools/breakdown.py --dtype f32 2>&1 | grep -E "solve|l=[56]"
done >> gpurun_out/ab_split.txt 2>&1
