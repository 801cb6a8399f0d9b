set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_next.py tests/test_gpu_multirank.py -m gpu -q -x -p no:cacheprovider -k "bicgstabl or next3 or sharded_cfg1 or cluster" > gpurun_out/pytest_bl.log 2>&1; echo pytest=$?; tail -30 gpurun_out/pytest_bl.log
timeout 900 python tools/bench_all.py --configs 1,2,3,5,4 --no-dense4 --methods bicgstabl > gpurun_out/bench_bl.log 2>&1; echo b=$?; cut -c1-220 gpurun_out/bench_bl.log
