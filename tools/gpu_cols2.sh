set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_apply.py tests/test_gpu_solve.py tests/test_gpu_next.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_cols2.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_cols2.log
timeout 900 python tools/bench_all.py --configs 2 > gpurun_out/bench_cols2.log 2>&1; echo b=$?
