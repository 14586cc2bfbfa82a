# A/B: fused z-marching passes vs step kernels on the small SR boxes (SR_FMG_FUSED_MIN_E)
mkdir -p gpurun_out
for rep in 1 2; do for v in 0 15 23; do
  echo "== min_e=$v f64"; SR_FMG_FUSED_MIN_E=$v timeout 300 python tools/breakdown.py 2>&1 | grep -E "solve|l=[56]"
done; done > gpurun_out/ab_mine.txt 2>&1
for v in 0 15 23; do
  echo "== min_e=$v f32"; SR_FMG_FUSED_MIN_E=$v timeout 300 python tools/breakdown.py --dtype f32 2>&1 | grep -E "solve"
done >> gpurun_out/ab_mine.txt 2>&1
