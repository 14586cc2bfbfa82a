for m in 1 3; do
SR_FMG_PASS=$m timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launch_pass$m.csv python tools/ncu_solve.py --config C3 --what solve --graph 0 > gpurun_out/ncu_list$m.log 2>&1
done
