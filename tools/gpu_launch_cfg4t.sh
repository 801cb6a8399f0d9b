# config 4 FFT lattice operator: launch list (cold, serialised) of a COCR and a BiCGSTAB solve
set -x
mkdir -p gpurun_out/summ4
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__registers_per_thread --clock-control none --csv"
for m in cocr bicgstab; do
timeout 900 ncu $M -s 300 -c 80 --log-file gpurun_out/summ4/launches_cfg4t_$m.csv python tools/bench_all.py --configs 4 --no-dense4 --reps 1 --methods $m > /dev/null 2>&1; echo $m=$?
done
