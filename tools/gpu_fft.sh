set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_next.py tests/test_gpu_multirank.py -m gpu -q -x -p no:cacheprovider -k "toeplitz" > gpurun_out/pytest_fft.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_fft.log
timeout 900 python tools/bench_all.py --configs 2,4 --no-dense4 --methods bicgstab,qmr,cocr,gmres > gpurun_out/bench_fft.log 2>&1; echo b=$?
