set -x
mkdir -p gpurun_out
timeout 600 python tools/bench_all.py --configs 5 > gpurun_out/bench5.log 2>&1; echo b=$?; cut -c1-200 gpurun_out/bench5.log
CMD="python tools/bench_all.py --configs 5 --reps 1 --methods bicgstab"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"spmv_sell" -s 100 -c 1 -o gpurun_out/prof5s $CMD > gpurun_out/ncu5s.log 2>&1; echo ncu=$?
