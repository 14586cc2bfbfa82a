# A/B: fused up pass (correction + post-smoothing, SR_FMG_UP_FUSE=1) per level
mkdir -p gpurun_out
for dt in f64 f32; do
for v in 0 1 0 1; do
  echo "== up=$v $dt"; SR_FMG_UP_FUSE=$v timeout 300 python tools/breakdown.py --dtype $dt 2>&1 | grep -E "solve|l=[5678]" | grep -E "solve|cheb2|prolong|pass_up"
done
done > gpurun_out/ab_up.txt 2>&1
