set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_next.py tests/test_gpu_multirank.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_next3.log 2>&1; echo pytest=$?; tail -30 gpurun_out/pytest_next3.log
timeout 900 python tools/bench_all.py --configs 1,2,3 --methods bicg,cgs,cocr,cgnr > gpurun_out/next3_bench.log 2>&1; echo bench=$?; cat gpurun_out/next3_bench.log
