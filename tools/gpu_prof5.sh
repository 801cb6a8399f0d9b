set -x
mkdir -p gpurun_out
CMD="python tools/bench_all.py --configs 5 --reps 1 --methods bicgstab"
timeout 300 $CMD > gpurun_out/plain5.log 2>&1; echo plain=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 3000 -c 40 --csv --log-file gpurun_out/launches5.csv $CMD > gpurun_out/ncu5.log 2>&1; echo ncu5=$?
CMD4="python tools/bench_all.py --configs 4 --no-dense4 --reps 1 --methods bicgstab"
timeout 300 $CMD4 > gpurun_out/plain4.log 2>&1; echo plain4=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -s 200 -c 40 --csv --log-file gpurun_out/launches4.csv $CMD4 > gpurun_out/ncu4.log 2>&1; echo ncu4=$?
