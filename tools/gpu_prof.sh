set -x
mkdir -p gpurun_out
timeout 300 python tools/prof_kernels.py > gpurun_out/prof_plain.log 2>&1; echo plain=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"gemv_cols|gemv_n_split|gemv_h_stage1" -c 8 -o gpurun_out/prof_k python tools/prof_kernels.py > gpurun_out/prof_ncu.log 2>&1; echo ncu=$?
