set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_next.py -m gpu -q -x -p no:cacheprovider -k "gmres" > gpurun_out/pytest_gm.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gm.log
timeout 900 python tools/bench_all.py --configs 5,2 --methods gmres > gpurun_out/bench_gm.log 2>&1; echo b=$?
