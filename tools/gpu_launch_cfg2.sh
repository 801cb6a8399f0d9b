# config 2 dense launch lists (cold, serialised) for BiCGSTAB and QMR
set -x
mkdir -p gpurun_out/summ2
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none --csv"
for m in bicgstab qmr cocr; do
timeout 900 ncu $M -s 400 -c 100 --log-file gpurun_out/summ2/launches_cfg2_$m.csv python tools/bench_all.py --configs 2 --reps 2 --methods $m --ops2 dense > /dev/null 2>&1; echo $m=$?
done
timeout 300 python tools/bench_all.py --configs 2 --reps 20 --methods bicgstab,qmr,cocr --ops2 dense > gpurun_out/summ2/bench_cfg2.log 2>&1
