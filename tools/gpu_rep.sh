set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multirank.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_rep.log 2>&1; echo pytest=$?; tail -30 gpurun_out/pytest_rep.log
timeout 900 python -m pytest tests/test_gpu_apply.py tests/test_gpu_solve.py tests/test_gpu_next.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_rest.log 2>&1; echo pytest2=$?; tail -3 gpurun_out/pytest_rest.log
