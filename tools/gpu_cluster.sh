set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_next.py -m gpu -q -x -p no:cacheprovider -k "cluster" > gpurun_out/pytest_cluster.log 2>&1; echo pytest=$?; tail -30 gpurun_out/pytest_cluster.log
for c in 0 1; do CCG_CLUSTER=$c timeout 600 python tools/bench_all.py --configs 1 > gpurun_out/bench1_cl$c.log 2>&1; echo b$c=$?; cat gpurun_out/bench1_cl$c.log | cut -c1-200; done
