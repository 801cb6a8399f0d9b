set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_next.py tests/test_gpu_multirank.py -m gpu -q -x -p no:cacheprovider -k "jacobi" > gpurun_out/pytest_jac.log 2>&1; echo pytest=$?; tail -30 gpurun_out/pytest_jac.log
