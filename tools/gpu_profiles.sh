# ncu --set full captures of the dominant kernel of every operator / path (one launch each)
set -x
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $B > gpurun_out/plain_bench.log 2>&1; echo plain=$?
timeout 900 $NCU -k regex:gemv_n_split -s 4 -c 1 -o gpurun_out/prof_gemv $B > gpurun_out/ncu_a.log 2>&1; echo a=$?
timeout 900 $NCU -k regex:gemv_h_stage1 -s 4 -c 1 -o gpurun_out/prof_gemvh $B > gpurun_out/ncu_b.log 2>&1; echo b=$?
timeout 900 $NCU -k regex:"gemv_cols<float, 256, 1, 1, 1" -s 2 -c 1 -o gpurun_out/prof_dual python tools/bench_all.py --configs 3 --reps 1 --methods qmr > gpurun_out/ncu_c.log 2>&1; echo c=$?
timeout 900 $NCU -k regex:spmv_sell -s 20 -c 1 -o gpurun_out/prof_sell python tools/bench_all.py --configs 5 --reps 1 --methods cocr > gpurun_out/ncu_d.log 2>&1; echo d=$?
timeout 900 $NCU -k regex:stencil7 -s 20 -c 1 -o gpurun_out/prof_stencil python tools/bench_all.py --configs 5 --reps 1 --methods cocr > gpurun_out/ncu_e.log 2>&1; echo e=$?
timeout 900 $NCU -k regex:fft_z_mul -s 20 -c 1 -o gpurun_out/prof_fftz python tools/bench_all.py --configs 4 --no-dense4 --reps 1 --methods cocr > gpurun_out/ncu_f.log 2>&1; echo f=$?
timeout 900 $NCU -k regex:"pass_kernel<256, BsX" -s 20 -c 1 -o gpurun_out/prof_passbsx python tools/bench_all.py --configs 5 --reps 1 --methods bicgstab > gpurun_out/ncu_g.log 2>&1; echo g=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1; echo list=$?
# summarise on the box (the reports exceed the copy-back limit), keep text only
python tools/ncu_summary.py gpurun_out gpurun_out/summ > gpurun_out/summ.log 2>&1; echo summ=$?
for r in gpurun_out/prof_*.ncu-rep; do n=$(basename $r .ncu-rep); ncu -i $r --page source --csv --print-source sass > gpurun_out/summ/${n}_sass.csv 2>/dev/null; done
gzip -f gpurun_out/summ/*_sass.csv
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
