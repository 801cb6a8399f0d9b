set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_next.py -m gpu -q -x -p no:cacheprovider -k "cluster" > gpurun_out/pytest_cluster.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_cluster.log
CCG_CLUSTER=1 timeout 600 python tools/bench_all.py --configs 1 > gpurun_out/bench1_cl1.log 2>&1; echo b1=$?; cat gpurun_out/bench1_cl1.log | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches1.csv python tools/bench_all.py --configs 1 --reps 3 --methods bicgstab,cgne > /dev/null 2>&1; echo ncu=$?
