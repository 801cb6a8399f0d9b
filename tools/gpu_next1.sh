# NEXT-1 check: new parity tests, cols vs split A·x sweep, QMR dual on/off throughput
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_next.py tests/test_gpu_solve.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_next.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_next.log
timeout 600 python tools/sweep_gemv.py --modes > gpurun_out/sweep_modes.log 2>&1; echo sweep=$?; cat gpurun_out/sweep_modes.log | tail -20
for d in 0 1; do CCG_QMR_DUAL=$d timeout 600 python tools/bench_all.py --configs 2,3 --methods qmr > gpurun_out/qmr_dual$d.log 2>&1; echo qmr$d=$?; cat gpurun_out/qmr_dual$d.log; done
CCG_GEMV=cols timeout 600 python tools/bench_all.py --configs 2,3 --methods bicgstab,cgne > gpurun_out/cols_bench.log 2>&1; echo cols=$?; cat gpurun_out/cols_bench.log
