# ncu --set full of the config 5 kernels after the load-ordering changes (one launch each), summarised on the box
set -x
mkdir -p gpurun_out/summ5b
NCU="ncu --set full --clock-control none --import-source on"
#timeout 900 $NCU -k regex:spmv_sell -s 20 -c 1 -o gpurun_out/prof_sell python tools/bench_all.py --configs 5 --reps 1 --methods cocr --ops csr > gpurun_out/summ5b/ncu_a.log 2>&1; echo a=$?
timeout 900 $NCU --kernel-name-base demangled -k regex:"ccg::BsX<double>>" -s 20 -c 1 -o gpurun_out/prof_passbsx python tools/bench_all.py --configs 5 --reps 1 --methods bicgstab --ops csr > gpurun_out/summ5b/ncu_b.log 2>&1; echo b=$?
python tools/ncu_summary.py gpurun_out gpurun_out/summ5b > gpurun_out/summ5b/summ.log 2>&1; echo summ=$?
for r in gpurun_out/prof_*.ncu-rep; do n=$(basename $r .ncu-rep); ncu -i $r --page details > gpurun_out/summ5b/${n}_details.txt 2>&1; done
rm -f gpurun_out/*.ncu-rep
