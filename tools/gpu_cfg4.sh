set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_solve.py -m gpu -q -x -p no:cacheprovider -k "cfg4" > gpurun_out/pytest_cfg4.log 2>&1; echo pytest=$?; tail -20 gpurun_out/pytest_cfg4.log
