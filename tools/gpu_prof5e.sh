set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_next.py tests/test_gpu_apply.py tests/test_gpu_solve.py -m gpu -q -x -p no:cacheprovider -k "csr or stencil" > gpurun_out/pytest_sell.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_sell.log
timeout 600 python tools/bench_all.py --configs 5 --methods bicgstab,cocr > gpurun_out/bench5.log 2>&1; echo b=$?; cut -c1-200 gpurun_out/bench5.log
