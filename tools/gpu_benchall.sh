set -x
mkdir -p gpurun_out
timeout 1500 python tools/bench_all.py --configs 1,2,3,5,4 > gpurun_out/bench_all.log 2>&1; echo bench=$?; cat gpurun_out/bench_all.log
