mkdir -p gpurun_out
CMD="python tools/bench_all.py --configs 5 --reps 1 --methods cors"
timeout 300 $CMD > gpurun_out/plain5.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 2000 -c 60 --csv --log-file gpurun_out/launches5.csv $CMD > gpurun_out/ncu5.log 2>&1; echo ncu=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_csr -s 50 -c 1 -o gpurun_out/prof_spmv $CMD > gpurun_out/ncu5f.log 2>&1; echo ncu=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:CoH -s 50 -c 1 -o gpurun_out/prof_pass $CMD > gpurun_out/ncu5p.log 2>&1; echo ncu=$?
