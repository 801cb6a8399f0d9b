set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_next.py -m gpu -q -x -p no:cacheprovider -k "callback" > gpurun_out/pytest_cb.log 2>&1; echo pytest=$?; tail -30 gpurun_out/pytest_cb.log
