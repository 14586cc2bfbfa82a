# coarse executor: per-op SM cycles and breakdowns for tiny thresholds 512 (default), 4096, 32768
mkdir -p gpurun_out
for t in 512 4096 32768; do
SR_FMG_CEXEC_TINY=$t timeout 120 python tools/cexec_prof.py > gpurun_out/cyt${t}.log 2> gpurun_out/cyt${t}.err
SR_FMG_CEXEC_TINY=$t timeout 300 python tools/breakdown.py > gpurun_out/bd_t${t}.txt 2>&1
done
