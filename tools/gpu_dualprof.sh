set -x
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,launch__registers_per_thread --clock-control none -k regex:gemv_cols -c 3 --csv python tools/prof_kernels.py > gpurun_out/dual_metrics.csv 2>gpurun_out/dual_err.log; echo ncu=$?
