set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_next.py tests/test_gpu_solve.py -m gpu -q -x -p no:cacheprovider -k "qmr or bicg or cols" > gpurun_out/pytest_ffma2.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_ffma2.log
timeout 900 python tools/bench_all.py --configs 3,2 --methods qmr,bicg > gpurun_out/bench_ffma2.log 2>&1; echo b=$?
