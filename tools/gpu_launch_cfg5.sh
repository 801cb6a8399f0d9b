# config 5 launch lists (cold, serialised; DRAM bytes per launch) for CSR BiCGSTAB / COCR and stencil COCR
set -x
mkdir -p gpurun_out/summ5
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none --csv"
timeout 900 ncu $M -s 3000 -c 120 --log-file gpurun_out/summ5/launches_csr_bicgstab${TAG}.csv python tools/bench_all.py --configs 5 --reps 1 --methods bicgstab --ops csr > /dev/null 2>&1; echo l1=$?
timeout 900 ncu $M -s 3000 -c 120 --log-file gpurun_out/summ5/launches_csr_cocr${TAG}.csv python tools/bench_all.py --configs 5 --reps 1 --methods cocr --ops csr > /dev/null 2>&1; echo l2=$?
timeout 900 ncu $M -s 3000 -c 120 --log-file gpurun_out/summ5/launches_st_cocr${TAG}.csv python tools/bench_all.py --configs 5 --reps 1 --methods cocr --ops stencil > /dev/null 2>&1; echo l3=$?
