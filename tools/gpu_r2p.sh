mkdir -p gpurun_out
for dt in f64 f32; do
for u in 1 2; do SR_FMG_RESTRICT_UNROLL=$u timeout 200 python tools/breakdown.py --dtype $dt > gpurun_out/bdp_${dt}_u$u.txt 2>&1; done
SR_FMG_RESTRICT_UNROLL=2 SR_FMG_RESTRICT_MINB=3 timeout 200 python tools/breakdown.py --dtype $dt > gpurun_out/bdp_${dt}_u2m3.txt 2>&1
done
