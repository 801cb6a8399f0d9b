# config 5 (CSR + stencil): per-kernel launch list with DRAM bytes, and full captures of the SELL SpMV per load schedule
set -x
mkdir -p gpurun_out/summ5
NCU="ncu --set full --clock-control none --import-source on"
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none --csv"
timeout 900 ncu $M -s 3000 -c 120 --log-file gpurun_out/summ5/launches_csr_bicgstab.csv python tools/bench_all.py --configs 5 --reps 1 --methods bicgstab > gpurun_out/summ5/l1.log 2>&1; echo l1=$?
timeout 900 ncu $M -s 3000 -c 120 --log-file gpurun_out/summ5/launches_csr_cocr.csv python tools/bench_all.py --configs 5 --reps 1 --methods cocr > gpurun_out/summ5/l2.log 2>&1; echo l2=$?
for m in 0 1; do
CCG_SELL_MODE=$m timeout 900 $NCU -k regex:spmv_sell -s 20 -c 1 -o gpurun_out/prof_sell_m$m python tools/bench_all.py --configs 5 --reps 1 --methods cocr > gpurun_out/summ5/ncu_m$m.log 2>&1; echo m$m=$?
ncu -i gpurun_out/prof_sell_m$m.ncu-rep --page details > gpurun_out/summ5/prof_sell_m${m}_details.txt 2>&1
ncu -i gpurun_out/prof_sell_m$m.ncu-rep --page raw --csv > gpurun_out/summ5/prof_sell_m${m}_raw.csv 2>&1
done
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
