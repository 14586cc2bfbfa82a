# knob sweep: prolongation rows per thread / band height, restriction unroll (fp64, fp32)
mkdir -p gpurun_out
for dt in f64 f32; do
  timeout 200 python tools/breakdown.py --dtype $dt > gpurun_out/bdm_${dt}_base.txt 2>&1
  SR_FMG_PROLONG_MAXS=6 timeout 200 python tools/breakdown.py --dtype $dt > gpurun_out/bdm_${dt}_pm6.txt 2>&1
  SR_FMG_PROLONG_MAXS=6 SR_FMG_PROLONG_BH=24 timeout 200 python tools/breakdown.py --dtype $dt > gpurun_out/bdm_${dt}_pm6b24.txt 2>&1
  SR_FMG_RESTRICT_UNROLL=2 timeout 200 python tools/breakdown.py --dtype $dt > gpurun_out/bdm_${dt}_ru2.txt 2>&1
done
