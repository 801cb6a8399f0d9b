set -x
mkdir -p gpurun_out
CMD="python tools/bench_all.py --configs 5 --reps 1 --methods bicgstab"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"BsX|spmv_sell_kernel" -s 200 -c 2 -o gpurun_out/prof5 $CMD > gpurun_out/ncu5b.log 2>&1; echo ncu=$?
