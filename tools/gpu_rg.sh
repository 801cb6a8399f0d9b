set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_next.py -m gpu -q -x -p no:cacheprovider -k "cols or qmr or bicg" > gpurun_out/pytest_rg.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_rg.log
timeout 900 python tools/sweep_gemv.py --modes > gpurun_out/sweep_rg.log 2>&1; echo sweep=$?; cat gpurun_out/sweep_rg.log
timeout 900 python tools/bench_all.py --configs 2,3,4 --methods qmr,bicg > gpurun_out/dual_s.log 2>&1; echo b=$?; cat gpurun_out/dual_s.log
